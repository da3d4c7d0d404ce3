# coarse levels: one 10-sweep segment per warp iteration when its regions fit one wave
set -u
O=gpurun_out
STITCH_B200_HS_COARSE1=1 python -m pytest tests/test_ref_pin.py tests/test_gpu_parity.py -m gpu -q -x -k "not variants" > $O/e25_tests.log 2>&1; echo "coarse1 tests rc=$?"
for rep in 1 2; do for c in 0 1; do
  STITCH_B200_HS_COARSE1=$c python bench.py --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 50 > $O/e25_c$c.json 2> $O/e25_c$c.err
  python -c "import json;d=json.loads(open('$O/e25_c$c.json').read().strip().splitlines()[-1]);k=d['kernels'];print('coarse1=$c', d['value'], d['e2e']['value'], d['p50_ms_per_frame'], k['hs_sweeps']['ms_per_frame'], d['kernels_per_frame'])"
done; done
