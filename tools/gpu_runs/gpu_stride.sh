set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/stride_pytest.log
timeout 1200 python bench.py > gpurun_out/stride_bench.log 2>&1
exit 0
