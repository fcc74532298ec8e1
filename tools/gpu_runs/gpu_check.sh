# engine + prefill parity tests, then a short decode bench
set -x
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_prefill.py -x -q 2>&1 | tail -5 > gpurun_out/pytest_engine.log || exit 3
timeout 600 python bench.py --steps 3 --warmup 3 --no-prefill --no-cpu --e2e-steps 0 > gpurun_out/bench_quick.log 2>&1
exit 0
