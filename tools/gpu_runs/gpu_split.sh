set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/split_pytest.log
timeout 900 python bench.py --steps 5 --no-cpu --e2e-steps 2 --no-prefill > gpurun_out/split_bench.log 2>&1
timeout 300 python tools/profile_kernels.py timeline 64 > gpurun_out/split_tl.log 2>&1
timeout 300 python tools/profile_kernels.py allhit 64 > gpurun_out/split_allhit.log 2>&1
exit 0
