#!/bin/bash
# One gpurun call: GPU parity suite, smoke, default bench, ncu launch list of the
# bench, ncu --set full of the top kernels. Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 0 --iters 50 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 40 -c 2 \
    -o gpurun_out/scan_full -f python tools/profile_run.py 64 30 > gpurun_out/ncu_scan.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:counts_kernel -c 1 \
    -o gpurun_out/counts_full -f python tools/profile_run.py 1 2 > gpurun_out/ncu_counts.log 2>&1
echo done
