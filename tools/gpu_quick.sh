#!/bin/bash
# Quick check of a walk-kernel change: GPU parity suite + a short bench line
# (+ optional ncu of the walk kernel with source). Outputs gpurun_out/$1/.
set -u
D=gpurun_out/${1:-q}; mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -q -x > $D/pytest_gpu.log 2>&1; echo "rc=$?" >> $D/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-extras --parity-chains 16 > $D/bench.json 2> $D/bench.err
if [ "${2:-}" = ncu ]; then
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:walk_chain -s 2 -c 1 \
    -o $D/walk_bench -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extras --parity-chains 0 > $D/ncu_walk.log 2>&1
cp paper_1210_5128_b200/libbnmc_b200.so $D/lib_snapshot.so
fi
echo done
