set -x
nvidia-smi -L
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r2_pytest_gpu0.log
timeout 600 python bench.py > gpurun_out/r2_bench0.log 2>&1
exit 0
