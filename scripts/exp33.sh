# programmatic dependent launch between a frame's kernels (STITCH_B200_PDL 0 / 1 / 2)
set -u
O=gpurun_out
for m in 1 2; do STITCH_B200_PDL=$m timeout 900 python -m pytest tests/test_ref_pin.py tests/test_gpu_parity.py -m gpu -q -x -k "not variants" > $O/e33_p${m}_tests.log 2>&1; echo "pdl=$m tests rc=$?"; tail -1 $O/e33_p${m}_tests.log; done
for rep in 1 2; do for m in 0 1 2; do
  STITCH_B200_PDL=$m timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 100 > $O/e33_p$m.json 2> $O/e33_p$m.err
  python -c "import json;d=json.loads(open('$O/e33_p$m.json').read().strip().splitlines()[-1]);print('pdl=$m', d['value'], d['e2e']['value'], d['p50_ms_per_frame'])"
done; done
