#!/bin/bash
# Launch list + one ncu --set full capture of the MTI pass of a config; exports the raw metrics and
# the per-line source page as CSV (the .ncu-rep itself stays on the box when it is large).
# usage: tools/ncu_capture.sh <config> <tag> <kernel-regex> [skip-launches] [extra bench args]
CFG=${1:-c3}; TAG=${2:-r2}; KRE=${3:-"k_walk"}; SKIP=${4:-8}; shift 4; EXTRA="$@"
CMD="python bench.py --config $CFG --steps 9 --warmup 3 --no-e2e --no-cpu-baseline $EXTRA"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_${CFG}_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}_${TAG}.csv $CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s $SKIP -c 1 -o /tmp/prof_${CFG}_${TAG} $CMD > gpurun_out/ncu_full_${CFG}_${TAG}.log 2>&1
echo "rc=$?"
ncu -i /tmp/prof_${CFG}_${TAG}.ncu-rep --page raw --csv > gpurun_out/raw_${CFG}_${TAG}.csv 2>/dev/null
ncu -i /tmp/prof_${CFG}_${TAG}.ncu-rep --page source --print-source cuda,sass --csv 2>/dev/null | gzip > gpurun_out/src_${CFG}_${TAG}.csv.gz
ls -la /tmp/prof_${CFG}_${TAG}.ncu-rep; S=$(stat -c %s /tmp/prof_${CFG}_${TAG}.ncu-rep); if [ "$S" -lt 40000000 ]; then cp /tmp/prof_${CFG}_${TAG}.ncu-rep gpurun_out/; fi
