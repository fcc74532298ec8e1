set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/cnt_pytest.log
timeout 900 python bench.py --steps 5 --no-cpu --e2e-steps 2 --no-regimes > gpurun_out/cnt_bench.log 2>&1
exit 0
