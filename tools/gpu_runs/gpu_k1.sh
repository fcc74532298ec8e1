# K1 change gate: engine parity tests + allhit profile (K1 phase stamps) + short bench
set -x
timeout 600 python -m pytest tests/test_gpu_engine.py -x -q 2>&1 | tail -3 > gpurun_out/pytest_engine.log || exit 3
timeout 300 python tools/profile_kernels.py allhit 64 > gpurun_out/allhit.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-prefill --no-cpu --e2e-steps 0 > gpurun_out/bench_quick.log 2>&1
exit 0
