set -x
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_prefill.py tests/test_gpu_parity_big.py -x -q 2>&1 | tail -5 > gpurun_out/od_pytest.log
timeout 300 python tools/profile_kernels.py timeline 64 > gpurun_out/od_tl.log 2>&1
timeout 900 python bench.py --steps 5 --no-cpu --e2e-steps 2 --no-regimes > gpurun_out/od_bench.log 2>&1
exit 0
