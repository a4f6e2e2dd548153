#!/bin/bash
# Profile the MTI assign kernel of the bench workload (one launch, iteration ~12) and the
# launch list of a short bench run.  Usage: tools/ncu_assign.sh <config> <tag>
CFG=${1:-c3}; TAG=${2:-r1}
CMD="python bench.py --config $CFG --steps 9 --warmup 3 --no-e2e --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$CFG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}_${TAG}.csv $CMD > gpurun_out/ncu_launches_$CFG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_assign|k_mti_tc" -s 10 -c 1 -o gpurun_out/prof_${CFG}_${TAG} $CMD > gpurun_out/ncu_full_$CFG.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/ncu_full_$CFG.log
