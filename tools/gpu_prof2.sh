#!/bin/bash
set -u
mkdir -p gpurun_out
make -s -C tests/cxx > gpurun_out/cxx_build.log 2>&1
timeout 600 ./tests/cxx/_build/test_dropin gpu > gpurun_out/cxx_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/cxx_gpu.log
for C in 1 64; do
  timeout 120 python tools/bench_scan_one.py $C 20 40 50 >> gpurun_out/scan_one.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 1 -c 1 \
    -o gpurun_out/scan_c64 -f python tools/bench_scan_one.py 64 20 40 2 > gpurun_out/ncu_scan64.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 1 -c 1 \
    -o gpurun_out/scan_c1 -f python tools/bench_scan_one.py 1 20 40 2 > gpurun_out/ncu_scan1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_kernel -c 1 \
    -o gpurun_out/k1_full -f python tools/profile_run.py 1 2 > gpurun_out/ncu_k1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 20 -c 1 \
    -o gpurun_out/step_c64 -f python tools/profile_run.py 64 40 > gpurun_out/ncu_step.log 2>&1
echo done
