#!/bin/bash
# Round evidence in one gpurun call: GPU parity suite, smoke, default bench,
# reference arm, ncu launch list of a short bench, ncu --set full of the
# headline walk kernel (bench config) and of K1. Outputs under gpurun_out/ev/.
set -u
D=gpurun_out/ev; mkdir -p $D
nvidia-smi > $D/nvidia_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err
timeout 900 python bench.py --impl reference > $D/bench_ref.json 2> $D/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras > $D/bench_ncu.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:walk_chain -s 2 -c 1 \
    -o $D/walk_bench -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extras > $D/ncu_walk.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_kernel -c 1 \
    -o $D/k1 -f python tools/profile_run.py 1 2 > $D/ncu_k1.log 2>&1
echo done
