# balance LUT: last-CTA election in the canvas (0) vs its own launch (1)
set -u
O=gpurun_out
STITCH_B200_CANVAS_SPLIT=1 python -m pytest tests/test_ref_pin.py tests/test_gpu_parity.py -m gpu -q -x -k "not variants" > $O/e24_tests.log 2>&1; echo "split tests rc=$?"
for rep in 1 2; do for sp in 0 1; do
  STITCH_B200_CANVAS_SPLIT=$sp python bench.py --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 50 > $O/e24_s$sp.json 2> $O/e24_s$sp.err
  python -c "import json;d=json.loads(open('$O/e24_s$sp.json').read().strip().splitlines()[-1]);k=d['kernels'];print('split=$sp', d['value'], d['e2e']['value'], d['p50_ms_per_frame'], k['canvas_balance']['ms_per_frame'], d['kernels_per_frame'])"
done; done
