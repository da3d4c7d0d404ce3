# Sweep variants: where the per-pixel denominator / reciprocal come from
# (record of a measurement: the exp_so/ builds it swapped in were local, git-ignored and are gone; rebuild with the EXTRA= flags named in DESIGN.md §4 to repeat it)
# (HS_YSMEM 0 / 1 / 2, prebuilt under exp_so/ys*/).  Parity subset + bench.
set -u
O=gpurun_out
P=paper_2308_09209_b200
for v in 0 1 2; do
  cp exp_so/ys$v/libstitch_b200.so $P/libstitch_b200.so
  python -m pytest tests/test_ref_pin.py tests/test_gpu_parity.py -m gpu -q -x > $O/e13_ys${v}_tests.log 2>&1; echo "ys$v tests rc=$?"
  python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 50 > $O/e13_ys${v}_bench.json 2> $O/e13_ys${v}_bench.err; echo "ys$v bench rc=$?"
done
for v in 1 2 0; do
  cp exp_so/ys$v/libstitch_b200.so $P/libstitch_b200.so
  python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 50 > $O/e13_ys${v}_bench2.json 2> $O/e13_ys${v}_bench2.err; echo "ys$v bench2 rc=$?"
done
