set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2c_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/r2c_bench.log 2>&1
exit 0
