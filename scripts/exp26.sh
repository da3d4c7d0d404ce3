# crop warp: rows per thread 1 / 2 / 4
# (the STITCH_B200_CROP_RPT variant was removed after this measurement: no gain)
set -u
O=gpurun_out
for r in 2 4; do STITCH_B200_CROP_RPT=$r python -m pytest tests/test_ref_pin.py tests/test_gpu_parity.py -m gpu -q -x -k "not variants" > $O/e26_r${r}_tests.log 2>&1; echo "rpt=$r tests rc=$?"; done
for rep in 1 2; do for r in 1 2 4; do
  STITCH_B200_CROP_RPT=$r python bench.py --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 50 > $O/e26_r$r.json 2> $O/e26_r$r.err
  python -c "import json;d=json.loads(open('$O/e26_r$r.json').read().strip().splitlines()[-1]);k=d['kernels'];print('rpt=$r', d['value'], d['e2e']['value'], d['p50_ms_per_frame'], k['crop_warp']['ms_per_frame'])"
done; done
