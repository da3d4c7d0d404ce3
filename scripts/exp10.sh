set -u
O=gpurun_out
python -m pytest tests/test_ref_pin.py tests/test_golden.py tests/test_gpu_parity.py tests/test_gpu_files.py tests/test_integration_binding.py tests/test_cpp_api.py -m gpu -q > $O/e10_tests.log 2>&1; echo "tests rc=$?"
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 100 > $O/e10_bench.json 2> $O/e10_bench.err; echo "bench rc=$?"
