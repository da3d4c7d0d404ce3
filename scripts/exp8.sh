set -u
O=gpurun_out
python -m pytest tests/test_gpu_parity.py -q -k "pageable or pipelined or tickets" > $O/e8_tests.log 2>&1; echo "tests rc=$?"
python -m pytest tests/test_integration_binding.py -m gpu -q > $O/e8_int.log 2>&1; echo "int rc=$?"
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 200 > $O/e8_bench.json 2> $O/e8_bench.err; echo "bench rc=$?"
