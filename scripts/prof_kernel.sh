#!/bin/bash
# Usage: scripts/prof_kernel.sh <kernel-regex> <skip-launches> <out-name> [env...]
# Runs the short bench once plainly, then ncu --set full on one launch of the
# named kernel (B200_PROFILING.md recipe).  Outputs land in gpurun_out/.
set -u
K=$1; SKIP=$2; NAME=$3
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --frame-sets 2"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$NAME.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 \
    -o gpurun_out/$NAME $CMD > gpurun_out/ncu_$NAME.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_$NAME.log
