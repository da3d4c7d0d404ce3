# explicit early PDL trigger (griddepcontrol.launch_dependents before the final stores of
# (record of a measurement: the exp_so/ builds were local and are gone; PDL_TRIGGER is now on by default, -DPDL_TRIGGER=0 is the t0 build)
# the sweep segments and the linearisation): builds exp_so/t0 (none) and exp_so/t1
set -u
O=gpurun_out
P=paper_2308_09209_b200
cp exp_so/t1/libstitch_b200.so $P/libstitch_b200.so
timeout 900 python -m pytest tests/test_ref_pin.py tests/test_gpu_parity.py -m gpu -q -x -k "not variants" > $O/e34_tests.log 2>&1; echo "trigger tests rc=$?"; tail -1 $O/e34_tests.log
for rep in 1 2; do for v in t0 t1; do
  cp exp_so/$v/libstitch_b200.so $P/libstitch_b200.so
  timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 100 > $O/e34_$v.json 2> $O/e34_$v.err
  python -c "import json;d=json.loads(open('$O/e34_$v.json').read().strip().splitlines()[-1]);print('$v', d['value'], d['e2e']['value'], d['p50_ms_per_frame'])"
done; done
cp exp_so/t0/libstitch_b200.so $P/libstitch_b200.so
