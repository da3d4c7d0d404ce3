#!/bin/bash
# Usage: scripts/launch_list.sh <out-name> [bench args...]
# ncu launch list (gpu__time_duration per kernel, B200_PROFILING.md recipe) of
# a short bench run, after the same command exits 0 without ncu.
set -u
NAME=$1; shift
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --frame-sets 2 $*"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$NAME.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/$NAME.csv $CMD > gpurun_out/ncu_$NAME.log 2>&1
echo "launch list rc=$?"
