# quick K3 loop: microbench, kernel numerics + engine parity, sweep, profiling timeline
set -x
tools/bench/k3_mma_bench > gpurun_out/k3f_mma.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py tests/test_gpu_prefill.py -x -q 2>&1 | tail -25 > gpurun_out/k3f_pytest.log
timeout 300 python tools/profile_kernels.py k3sweep 50 > gpurun_out/k3f_sweep.log 2>&1
FATE_PROF=1 python -m paper_2502_12224_b200.build --force > gpurun_out/k3f_build.log 2>&1
K3_SPECS=${K3_SPECS:-qwen_bench_mix,int2x4,int4x4} timeout 300 python tools/profile_kernels.py k3prof 20 > gpurun_out/k3f_prof.log 2>&1
python -m paper_2502_12224_b200.build --force >> gpurun_out/k3f_build.log 2>&1
exit 0
