set -u
O=gpurun_out
B="python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 200"
$B > $O/e1_s4.json 2> $O/e1_s4.err; echo "s4 rc=$?"
STITCH_B200_SLOTS=6 $B > $O/e1_s6.json 2> $O/e1_s6.err; echo "s6 rc=$?"
STITCH_B200_SLOTS=8 $B > $O/e1_s8.json 2> $O/e1_s8.err; echo "s8 rc=$?"
STITCH_B200_COLOR_PPT=16 $B > $O/e1_p16.json 2> $O/e1_p16.err; echo "p16 rc=$?"
STITCH_B200_COLOR_PPT=32 $B > $O/e1_p32.json 2> $O/e1_p32.err; echo "p32 rc=$?"
STITCH_B200_COPY_THREADS=14 $B > $O/e1_ct14.json 2> $O/e1_ct14.err; echo "ct14 rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --frame-sets 2"
$CMD > $O/e1_plain.log 2>&1 || { echo "plain failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:k_pair_color -s 4 -c 2 \
    -o $O/e1_ncu_color $CMD > $O/e1_ncu_color.log 2>&1; echo "ncu color rc=$?"
