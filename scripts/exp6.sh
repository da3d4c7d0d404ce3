set -u
O=gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_bench_path.py tests/test_ref_pin.py -m gpu -q -x > $O/e6_tests.log 2>&1; echo "tests rc=$?"
B="python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 100"
$B > $O/e6_rp.json 2> $O/e6_rp.err; echo "rp rc=$?"
STITCH_B200_HS_RP=0 $B > $O/e6_norp.json 2> $O/e6_norp.err; echo "norp rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --frame-sets 2"
$CMD > $O/e6_plain.log 2>&1 || { echo "plain failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:k_hs_sweep_rp -s 10 -c 1 \
    -o $O/e6_ncu_rp $CMD > $O/e6_ncu_rp.log 2>&1; echo "ncu rp rc=$?"
