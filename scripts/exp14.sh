# Paired-column sweep (STITCH_B200_HS_PAIR=1, default) vs the one-column
# layout (=0): parity subset + bench, interleaved.
set -u
O=gpurun_out
python -m pytest tests/test_ref_pin.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > $O/e14_tests.log 2>&1; echo "tests rc=$?"
for p in 1 0 1 0; do
  STITCH_B200_HS_PAIR=$p python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 50 > $O/e14_p${p}_bench.json 2> $O/e14_p${p}_bench.err; echo "p$p bench rc=$?"
  python -c "import json;d=json.loads(open('$O/e14_p${p}_bench.json').read().strip().splitlines()[-1]);print('p$p', d['value'], d['e2e']['value'])"
done
