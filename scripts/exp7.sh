set -u
O=gpurun_out
B="python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 100"
STITCH_B200_WARP_F32=1 $B > $O/e7_f32.json 2> $O/e7_f32.err; echo "f32 rc=$?"
$B > $O/e7_base.json 2> $O/e7_base.err; echo "base rc=$?"
CONTRACT_ENV=STITCH_B200_WARP_F32=1 python -m pytest scripts/fast_sweep_contract.py -q -s > $O/e7_contract.log 2>&1; echo "contract rc=$?"
