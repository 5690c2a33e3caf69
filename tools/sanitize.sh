#!/bin/bash
# compute-sanitizer evidence: racecheck / synccheck / memcheck over every kernel
# family (tools/sanitize_run.py). Logs under gpurun_out/san/.
set -u
D=gpurun_out/san; mkdir -p $D
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in ${SAN_TOOLS:-memcheck racecheck synccheck}; do
  for c in ${SAN_CASES:-k1 wide multi walk1 walk8 walk32 spec scan recheck}; do
    extra=""
    [ $tool = memcheck ] && extra="--leak-check full"
    [ $tool = racecheck ] && extra="--racecheck-report all"
    timeout 600 $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_run.py $c > $D/${tool}_$c.log 2>&1
    echo "$tool $c rc=$?" | tee -a $D/summary.txt
  done
done
