# K3 quick: sweep + profiling-build timeline (no tests)
set -x
timeout 300 python tools/profile_kernels.py k3sweep 50 > gpurun_out/k3iter_sweep.log 2>&1
FATE_PROF=1 python -m paper_2502_12224_b200.build --force > gpurun_out/k3prof_build.log 2>&1
K3_SPECS=qwen_bench_mix,int4x4 timeout 300 python tools/profile_kernels.py k3prof 20 > gpurun_out/k3prof.log 2>&1
exit 0
