set -x
timeout 1500 python -m pytest tests/test_gpu_parity_big.py -x -q --durations=10 2>&1 | tail -40 > gpurun_out/r2f_pytest.log
exit 0
