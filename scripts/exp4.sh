set -u
O=gpurun_out
python -m pytest tests/test_ref_pin.py tests/test_golden.py tests/test_gpu_parity.py -m gpu -q -x > $O/e4_tests.log 2>&1; echo "tests rc=$?"
B="python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 200"
$B > $O/e4_bench.json 2> $O/e4_bench.err; echo "bench rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --frame-sets 2"
$CMD > $O/e4_plain.log 2>&1 || { echo "plain failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:k_pair_color -s 4 -c 2 \
    -o $O/e4_ncu_color $CMD > $O/e4_ncu_color.log 2>&1; echo "ncu color rc=$?"
