set -x
timeout 300 python tools/profile_kernels.py k3sweep 50 > gpurun_out/k3sw.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 1 --no-prefill > gpurun_out/k3sw_bench.log 2>&1
exit 0
