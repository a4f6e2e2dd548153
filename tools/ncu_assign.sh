#!/bin/bash
# Profile the MTI assignment kernel of the bench workload: the launch list of a short bench run
# (gpu__time_duration, cold-cache serialised) and one --set full capture of the engine kernel
# at iteration ~12.  Usage: tools/ncu_assign.sh <config> <tag> <kernel-regex>
CFG=${1:-c3}; TAG=${2:-r1}; KRE=${3:-"k_walk|k_mti_tc|k_assign"}
CMD="python bench.py --config $CFG --steps 9 --warmup 3 --no-e2e --no-cpu-baseline"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$CFG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}_${TAG}.csv $CMD > gpurun_out/ncu_launches_$CFG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 8 -c 1 -o gpurun_out/prof_${CFG}_${TAG} $CMD > gpurun_out/ncu_full_$CFG.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/ncu_full_$CFG.log
