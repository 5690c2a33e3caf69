#!/bin/bash
mkdir -p gpurun_out/s2
timeout 900 python -m pytest tests -m gpu -x -q -k "mode or tie or chains or orders or scan or cfg4 or upload or refold or multi" > gpurun_out/s2/pytest.log 2>&1; tail -2 gpurun_out/s2/pytest.log
for C in 1 8 64; do timeout 120 python tools/bench_scan_one.py $C 20 40 50; done
for C in 1 64; do timeout 120 python tools/bench_scan_one.py $C 0 59 50; done
TW=8 timeout 300 python tools/walk_probe.py cfg4 200 1 2>&1 | grep "mode 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan2 -s 1 -c 1 \
    -o gpurun_out/s2/scan2_c1 -f python tools/bench_scan_one.py 1 0 59 2 > gpurun_out/s2/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan2 -s 1 -c 1 \
    -o gpurun_out/s2/scan2_c64 -f python tools/bench_scan_one.py 64 20 40 2 > gpurun_out/s2/ncu64.log 2>&1
