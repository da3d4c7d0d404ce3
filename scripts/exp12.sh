set -u
O=gpurun_out
python -m pytest tests/test_ref_pin.py tests/test_golden.py tests/test_gpu_parity.py tests/test_integration_binding.py tests/test_gpu_files.py -m gpu -q > $O/e12_tests.log 2>&1; echo "tests rc=$?"
python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 100 > $O/e12_bench.json 2> $O/e12_bench.err; echo "bench rc=$?"
python scripts/parity_report.py $O/r02_parity_report.json > $O/e12_parity.log 2>&1; echo "parity rc=$?"
