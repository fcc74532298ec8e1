set -x
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_parity_big.py -k "prefill or dsk" -x -q 2>&1 | tail -15 > gpurun_out/k4_pytest.log
timeout 600 python tools/profile_kernels.py prefill 512 > gpurun_out/k4_prefill.log 2>&1
exit 0
