#!/bin/bash
# One measurement pass for profiles/ (run under gpurun on one B200):
#   the default bench line (with the CPU baseline), BASELINE configs c1 / c3 /
#   c4 / c5 (64 streams on this GPU), the reference arm (c2: the port + the
#   c1 reference/port ratio; c1: the reference itself), the launch list with
#   DRAM bytes of every kernel, and ncu --set full captures of the level-0
#   Jacobi segment, the level-0 linearisation, the canvas kernel, the colour
#   statistics and the crop warp.  Each ncu run follows the same command
#   exiting 0 without ncu.  Outputs: gpurun_out/<tag>_*.
set -u
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?"
python bench.py --config c1 --no-cpu-baseline > $O/${TAG}_bench_c1.json 2> $O/${TAG}_bench_c1.err; echo "c1 rc=$?"
python bench.py --config c3 --no-cpu-baseline > $O/${TAG}_bench_c3.json 2> $O/${TAG}_bench_c3.err; echo "c3 rc=$?"
python bench.py --config c4 --no-cpu-baseline --steps 100 --e2e-steps 50 > $O/${TAG}_bench_c4.json 2> $O/${TAG}_bench_c4.err; echo "c4 rc=$?"
python bench.py --config c5 --no-cpu-baseline --steps 20 --e2e-steps 50 --frame-sets 4 > $O/${TAG}_bench_c5.json 2> $O/${TAG}_bench_c5.err; echo "c5 rc=$?"
python bench.py --impl reference --steps 20 --warmup 5 > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err; echo "reference rc=$?"
python bench.py --impl reference --config c1 --steps 20 --warmup 2 > $O/${TAG}_bench_ref_c1.json 2> $O/${TAG}_bench_ref_c1.err; echo "reference c1 rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --frame-sets 2"
$CMD > $O/${TAG}_plain.log 2>&1 || { echo "plain failed"; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file $O/${TAG}_launches.csv $CMD > $O/${TAG}_ncu_launches.log 2>&1; echo "launch list rc=$?"
# per frame the first 30 Jacobi launches are the coarse levels; launch 31 is
# the first level-0 segment (64 x 64 regions)
ncu --set full --clock-control none --import-source on -k regex:k_hs_sweep -s 30 -c 1 \
    -o $O/${TAG}_ncu_sweep $CMD > $O/${TAG}_ncu_sweep.log 2>&1; echo "ncu sweep rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_hs_linearize -s 6 -c 1 \
    -o $O/${TAG}_ncu_lin $CMD > $O/${TAG}_ncu_lin.log 2>&1; echo "ncu lin rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_canvas -s 2 -c 1 \
    -o $O/${TAG}_ncu_canvas $CMD > $O/${TAG}_ncu_canvas.log 2>&1; echo "ncu canvas rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_pair_color -s 4 -c 2 \
    -o $O/${TAG}_ncu_color $CMD > $O/${TAG}_ncu_color.log 2>&1; echo "ncu color rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_crop_warp -s 2 -c 1 \
    -o $O/${TAG}_ncu_crop $CMD > $O/${TAG}_ncu_crop.log 2>&1; echo "ncu crop rc=$?"
