#!/bin/bash
# One gpurun call of round evidence. Usage: bash tools/gpu_round.sh TAG [parts...]
# parts: tests fulltests bench dist ncu launches san (default: all)
set -u
TAG=$1; shift
PARTS=${*:-"tests bench dist launches ncu san"}
D=gpurun_out/$TAG; mkdir -p $D
nvidia-smi > $D/smi.txt 2>&1
for p in $PARTS; do case $p in
tests) timeout 1500 python -m pytest tests -m gpu -q -x > $D/pytest_gpu.log 2>&1; echo "rc=$?" >> $D/pytest_gpu.log ;;
smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "rc=$?" >> $D/smoke.log ;;
bench) timeout 900 python bench.py > $D/bench.json 2> $D/bench.err ;;
ref) timeout 900 python bench.py --impl reference > $D/bench_ref.json 2> $D/bench_ref.err ;;
dist) timeout 600 python bench.py --force-dist --steps 2 --warmup 1 --no-extras --no-cpu-baseline --parity-chains 0 > $D/bench_dist.json 2> $D/bench_dist.err ;;
launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extras --parity-chains 0 > $D/bench_ncu.log 2>&1 ;;
ncu) timeout 1200 ncu --set full --clock-control none --import-source on -k regex:walk_chain -s 2 -c 1 \
    -o $D/walk_bench -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extras --parity-chains 0 > $D/ncu_walk.log 2>&1 ;;
ncuk1) timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_kernel -c 1 \
    -o $D/k1 -f python tools/profile_run.py 1 2 > $D/ncu_k1.log 2>&1 ;;
san) for tool in memcheck racecheck synccheck; do for c in wide multi; do
       timeout 600 compute-sanitizer --tool $tool --print-limit 30 --error-exitcode 9 python tools/sanitize_run.py $c > $D/san_${tool}_$c.log 2>&1
       echo "$tool $c rc=$?" >> $D/san_summary.txt; done; done ;;
esac; done
echo done
