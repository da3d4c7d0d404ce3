set -u
O=gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_integration_binding.py tests/test_gpu_files.py -m gpu -q -x > $O/e18_tests.log 2>&1; echo "tests rc=$?"; tail -1 $O/e18_tests.log
for i in 1 2; do
python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 100 > $O/e18_bench$i.json 2> $O/e18_bench$i.err
python -c "import json;d=json.loads(open('$O/e18_bench$i.json').read().strip().splitlines()[-1]);e=d['e2e'];print(d['value'], e['value'], e.get('pageable_value'), e.get('sync_process_value'), e.get('sync_pageable_value'))"
done
python bench.py --config c1 --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 100 > $O/e18_c1.json 2> $O/e18_c1.err
python -c "import json;d=json.loads(open('$O/e18_c1.json').read().strip().splitlines()[-1]);e=d['e2e'];print('c1', d['value'], e['value'], e.get('pageable_value'), e.get('sync_process_value'), e.get('sync_pageable_value'))"
