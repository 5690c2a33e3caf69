#!/bin/bash
# K2 scan A/B (cold L2 per launch) + ncu of the single-order full scan.
set -u
D=gpurun_out/${1:-s3}; mkdir -p $D
run() { for C in 1 8 64; do timeout 180 python tools/bench_scan_one.py $C 0 59 30 >> $D/ab.txt 2>&1; done; }
BNMC_SCAN_KERNEL=2 run
for v in "128,8,0" "64,8,0" "128,4,0" "256,4,0" "256,8,0" "128,8,1" "128,8,2"; do
  echo "scan4 $v" >> $D/ab.txt; BNMC_SCAN_KERNEL=4 BNMC_SCAN4=$v run
done
BNMC_SCAN_KERNEL=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan -s 1 -c 1 \
  -o $D/scan4_c1 -f python tools/bench_scan_one.py 1 0 59 2 > $D/ncu1_4.log 2>&1
BNMC_SCAN_KERNEL=4 timeout 900 python -m pytest tests -m gpu -q -x -k "scan or order or full or mode" > $D/pytest_scan4.log 2>&1; echo "rc=$?" >> $D/pytest_scan4.log
echo done
