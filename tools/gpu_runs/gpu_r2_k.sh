set -x
timeout 900 python bench.py --steps 5 --no-cpu --e2e-steps 1 --no-prefill > gpurun_out/r2k_bench.log 2>&1
exit 0
