# Last-CTA election fence: membar.sc (ELECT_FENCE=0), fence.acq_rel (1),
# (record of a measurement: the exp_so/ builds it swapped in were local, git-ignored and are gone; rebuild with the EXTRA= flags named in DESIGN.md §4 to repeat it)
# release atomic + acq_rel (2); prebuilt under exp_so/ef*/.
set -u
O=gpurun_out
P=paper_2308_09209_b200
for v in 1 2; do
  cp exp_so/ef$v/libstitch_b200.so $P/libstitch_b200.so
  python -m pytest tests/test_ref_pin.py tests/test_gpu_parity.py -m gpu -q -x -k "not variants" > $O/e15_ef${v}_tests.log 2>&1; echo "ef$v tests rc=$?"
done
for v in 0 1 2 0 1 2; do
  cp exp_so/ef$v/libstitch_b200.so $P/libstitch_b200.so
  python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 50 > $O/e15_ef${v}_bench.json 2> $O/e15_ef${v}_bench.err
  python -c "import json;d=json.loads(open('$O/e15_ef${v}_bench.json').read().strip().splitlines()[-1]);k=d['kernels'];print('ef$v', d['value'], d['e2e']['value'], k['pair_color']['ms_per_frame'], k['canvas_balance']['ms_per_frame'])"
done
cp exp_so/ef0/libstitch_b200.so $P/libstitch_b200.so
