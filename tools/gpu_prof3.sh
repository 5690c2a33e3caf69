#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_walk.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras > gpurun_out/bench_ncu_walk.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_chain -s 2 -c 1 \
    -o gpurun_out/walk_bench -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extras > gpurun_out/ncu_walk_bench.log 2>&1
tail -2 gpurun_out/ncu_walk_bench.log
timeout 900 python tools/walk_probe.py cfg5 200 4736,18944 > gpurun_out/walk_probe_cfg5.log 2>&1; cat gpurun_out/walk_probe_cfg5.log
