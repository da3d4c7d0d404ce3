# TMA-staged Jacobi constants in the plain 64 x 64 segments (STITCH_B200_HS_TMA)
set -u
O=gpurun_out
STITCH_B200_HS_TMA=1 timeout 900 python -m pytest tests/test_ref_pin.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "not variants" > $O/e30_tests.log 2>&1; echo "tma tests rc=$?"; tail -2 $O/e30_tests.log
for rep in 1 2; do for t in 0 1; do
  STITCH_B200_HS_TMA=$t timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 50 > $O/e30_t$t.json 2> $O/e30_t$t.err
  python -c "import json;d=json.loads(open('$O/e30_t$t.json').read().strip().splitlines()[-1]);k=d['kernels'];print('tma=$t', d['value'], d['e2e']['value'], d['p50_ms_per_frame'], k['hs_sweeps']['ms_per_frame'])"
done; done
