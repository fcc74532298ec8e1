# K3 iteration: numerics + engine parity, then the profiling build's timeline and the sweep
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -x -q 2>&1 | tail -15 > gpurun_out/k3iter_pytest.log
timeout 300 python tools/profile_kernels.py k3sweep 50 > gpurun_out/k3iter_sweep.log 2>&1
FATE_PROF=1 python -m paper_2502_12224_b200.build --force > gpurun_out/k3prof_build.log 2>&1
timeout 300 python tools/profile_kernels.py k3prof 20 > gpurun_out/k3prof.log 2>&1
exit 0
