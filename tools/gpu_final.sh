#!/bin/bash
# Round evidence on one box: GPU parity suite, smoke, default bench, reference
# arm, ncu launch list, ncu --set full of the headline walk kernel and of K1,
# compute-sanitizer over every kernel family. Outputs under gpurun_out/$1/.
set -u
TAG=${1:-final}
bash tools/gpu_round.sh $TAG tests smoke bench ref launches ncu ncuk1
SAN_TOOLS="memcheck racecheck synccheck" bash tools/sanitize.sh
mkdir -p gpurun_out/$TAG/san && cp gpurun_out/san/* gpurun_out/$TAG/san/ 2>/dev/null
echo done
