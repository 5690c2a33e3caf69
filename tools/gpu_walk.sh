#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1; tail -3 gpurun_out/pytest_gpu3.log
timeout 600 python tools/walk_probe.py cfg4 500 ${CHAINS:-1,64,296,592,1184,2368,4736} > gpurun_out/walk_probe.log 2>&1; cat gpurun_out/walk_probe.log
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:walk_chain -c 1 \
    -o gpurun_out/walk_full -f python tools/walk_probe.py cfg4 100 592 > gpurun_out/ncu_walk.log 2>&1
tail -2 gpurun_out/ncu_walk.log
fi
