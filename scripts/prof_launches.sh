#!/bin/bash
# Launch list (per-kernel device time) of a short bench run, then one
# ncu --set full capture of the dominant kernel (B200_PROFILING.md recipe).
set -u
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 --frame-sets 2"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_launches.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
# dominant kernel: first level-0 sweep segment of the first frame
$CMD > gpurun_out/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_hs_sweep -s 30 -c 2 \
    -o gpurun_out/prof_sweep $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
