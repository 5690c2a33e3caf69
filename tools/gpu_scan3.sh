#!/bin/bash
# K2 scan A/B (cold L2 per launch) + ncu of the single-order full scan, then
# the walk bench line.
set -u
D=gpurun_out/${1:-s3}; mkdir -p $D
for v in "2 8,2,256" "3 8,2,256" "3 16,2,256"; do
  set -- $v
  for C in 1 8 64; do
    BNMC_SCAN_KERNEL=$1 BNMC_SCAN3=$2 timeout 180 python tools/bench_scan_one.py $C 0 59 30 >> $D/ab.txt 2>&1
  done
done
for K in 2 3; do
BNMC_SCAN_KERNEL=$K timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan -s 1 -c 1 \
  -o $D/scan${K}_c1 -f python tools/bench_scan_one.py 1 0 59 2 > $D/ncu1_$K.log 2>&1
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --parity-chains 0 > $D/bench.json 2> $D/bench.err
echo done
