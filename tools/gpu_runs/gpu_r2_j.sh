set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r2j_pytest.log
timeout 900 python bench.py > gpurun_out/r2j_bench.log 2>&1
timeout 600 python bench.py --no-dense --steps 3 --no-cpu --e2e-steps 1 --no-prefill > gpurun_out/r2j_bench_nodense.log 2>&1
timeout 300 python tools/profile_kernels.py timeline 64 > gpurun_out/r2j_timeline.log 2>&1
exit 0
