# frames in flight (pipeline slots) with the round-2 kernels: 3 / 4 / 5 / 6
set -u
O=gpurun_out
for rep in 1 2; do for n in 4 5 6 3; do
  STITCH_B200_SLOTS=$n timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 100 > $O/e31_s$n.json 2> $O/e31_s$n.err
  python -c "import json;d=json.loads(open('$O/e31_s$n.json').read().strip().splitlines()[-1]);print('slots=$n', d['value'], d['e2e']['value'], d['e2e']['pageable_value'], d['p50_ms_per_frame'])"
done; done
