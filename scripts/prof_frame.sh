#!/bin/bash
# Launch list of a short bench run plus one ncu --set full capture each of
# the canvas and level-0 linearisation kernels (B200_PROFILING.md recipe),
# each after the same command exits 0 without ncu.  Outputs in gpurun_out/.
set -u
TAG=${1:-cur}
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --frame-sets 2"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launches_$TAG.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:'k_canvas|k_hs_linearize' -s 8 -c 2 \
    -o gpurun_out/prof_canvas_lin_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
