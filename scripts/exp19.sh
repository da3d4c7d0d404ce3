set -u
O=gpurun_out
python -m pytest tests/test_ref_errors.py tests/test_ref_pin.py tests/test_gpu_parity.py tests/test_integration_binding.py tests/test_gpu_files.py tests/test_cpp_api.py -m gpu -q -x > $O/e19_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/e19_tests.log
python bench.py --steps 200 --warmup 5 --no-cpu-baseline --e2e-steps 100 > $O/e19_bench.json 2> $O/e19_bench.err
python -c "import json;d=json.loads(open('$O/e19_bench.json').read().strip().splitlines()[-1]);e=d['e2e'];print(d['value'], e['value'], e.get('pageable_value'), e.get('sync_process_value'), e.get('sync_pageable_value'))"
