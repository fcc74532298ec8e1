# prefill (K4 tcgen05) parity + numerics, then DSK prefill throughput
set -x
timeout 600 python -m pytest tests/test_gpu_prefill.py -x -q -s 2>&1 | tail -30 > gpurun_out/pytest_prefill.log || exit 3
timeout 600 python tools/profile_kernels.py prefill 512 > gpurun_out/prefill_perf.log 2>&1
exit 0
