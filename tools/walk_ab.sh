#!/bin/bash
# Same-box A/B of walk-kernel builds (tools/build_variant.sh) and settings:
# interleaved walk_probe runs at the bench configuration.
#   bash tools/walk_ab.sh OUT SPEC...   SPEC = VARIANT[:ENV=VALUE[,ENV=VALUE]]
set -u
OUT=gpurun_out/$1; shift; mkdir -p $OUT
for rep in 1 2 3; do
  for spec in "$@"; do
    v=${spec%%:*}; envs=""; [ "$spec" != "$v" ] && envs=$(echo "${spec#*:}" | tr ',' ' ')
    echo "== $spec rep $rep" >> $OUT/ab.txt
    env $envs BNMC_B200_LIB=variants/$v/libbnmc_b200.so timeout 300 python tools/walk_probe.py ${CFG:-cfg4} ${ITERS:-500} ${CHAINS:-18944} >> $OUT/ab.txt 2>&1
  done
done
echo done
