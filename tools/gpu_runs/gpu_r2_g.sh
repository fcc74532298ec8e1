# K3 iteration: numerics + engine parity, sweep, then the profiling build's timeline
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -x -q 2>&1 | tail -15 > gpurun_out/r2g_pytest.log
timeout 300 python tools/profile_kernels.py k3sweep 50 > gpurun_out/r2g_k3sweep.log 2>&1
FATE_PROF=1 python -m paper_2502_12224_b200.build --force > gpurun_out/r2g_build.log 2>&1
K3_SPECS=qwen_bench_mix,bf16_shared,int2x4,int4x4 timeout 300 python tools/profile_kernels.py k3prof 20 > gpurun_out/r2g_k3prof.log 2>&1
python -m paper_2502_12224_b200.build --force >> gpurun_out/r2g_build.log 2>&1
exit 0
