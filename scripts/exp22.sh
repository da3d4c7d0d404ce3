# 3D-M statistics variants: 16-byte loads (COLOR_VEC) x separate solve launch (COLOR_SPLIT)
set -u
O=gpurun_out
for cfg in "0 0" "1 0" "0 1" "1 1"; do
  set -- $cfg
  export STITCH_B200_COLOR_VEC=$1 STITCH_B200_COLOR_SPLIT=$2
  python -m pytest tests/test_ref_pin.py tests/test_gpu_parity.py -m gpu -q -x -k "not variants" > $O/e22_v$1s$2_tests.log 2>&1; echo "vec=$1 split=$2 tests rc=$?"
done
for rep in 1 2; do
for cfg in "0 0" "1 0" "0 1" "1 1"; do
  set -- $cfg
  export STITCH_B200_COLOR_VEC=$1 STITCH_B200_COLOR_SPLIT=$2
  python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 50 > $O/e22_v$1s$2_bench.json 2> $O/e22_v$1s$2_bench.err
  python -c "import json;d=json.loads(open('$O/e22_v$1s$2_bench.json').read().strip().splitlines()[-1]);k=d['kernels'];print('vec=$1 split=$2', d['value'], d['e2e']['value'], d['p50_ms_per_frame'], k['pair_color']['ms_per_frame'], d['kernels_per_frame'])"
done
done
