set -u
O=gpurun_out
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 100"
$B > $O/e9_a.json 2> $O/e9_a.err; echo "a rc=$?"
STITCH_B200_SYNC_DIRECT=1 $B > $O/e9_b.json 2> $O/e9_b.err; echo "b rc=$?"
STITCH_B200_COPY_THREADS=4 $B > $O/e9_c.json 2> $O/e9_c.err; echo "c rc=$?"
