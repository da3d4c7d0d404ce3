# balance LUT with the threshold history staged in shared memory
set -u
O=gpurun_out
python -m pytest tests/test_ref_pin.py tests/test_ref_errors.py tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x > $O/e29_tests.log 2>&1; echo "tests rc=$?"; tail -1 $O/e29_tests.log
for rep in 1 2; do
python bench.py --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 50 > $O/e29.json 2> $O/e29.err
python -c "import json;d=json.loads(open('$O/e29.json').read().strip().splitlines()[-1]);k=d['kernels'];print(d['value'], d['e2e']['value'], d['p50_ms_per_frame'], k['pair_color']['ms_per_frame'], k['canvas_balance']['ms_per_frame'])"
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --frame-sets 2"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_pair_solve|k_balance" -c 40 --csv --log-file $O/e29_launches.csv $CMD > /dev/null 2>&1; echo "ncu rc=$?"
