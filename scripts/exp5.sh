set -u
O=gpurun_out
python bench.py --config c3 --no-cpu-baseline > $O/r02_bench_c3.json 2> $O/r02_bench_c3.err; echo "c3 rc=$?"
B="python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 100"
STITCH_B200_WARP_STAGE=1 $B > $O/e5_stage.json 2> $O/e5_stage.err; echo "stage rc=$?"
$B > $O/e5_base.json 2> $O/e5_base.err; echo "base rc=$?"
python -m pytest tests/test_gpu_parity.py -q -k "WARP_STAGE" > $O/e5_stage_test.log 2>&1; echo "stage test rc=$?"
python -m pytest tests/test_integration_binding.py tests/test_bench_launcher.py -m gpu -q > $O/e5_int.log 2>&1; echo "int rc=$?"
