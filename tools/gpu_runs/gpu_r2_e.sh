# K3 evidence: per-format sweep, ncu full capture on the bench mix, then the profiling build's timeline
set -x
timeout 300 python tools/profile_kernels.py k3sweep 50 > gpurun_out/r2e_k3sweep.log 2>&1
K3_SPECS=qwen_bench_mix timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_kernel -s 6 -c 1 -o gpurun_out/r2e_k3_full python tools/profile_kernels.py k3prof 8 > gpurun_out/r2e_ncu.log 2>&1
FATE_PROF=1 python -m paper_2502_12224_b200.build --force > gpurun_out/r2e_build.log 2>&1
K3_SPECS=qwen_bench_mix,bf16_shared,int2x4,int4x4 timeout 300 python tools/profile_kernels.py k3prof 20 > gpurun_out/r2e_k3prof.log 2>&1
python -m paper_2502_12224_b200.build --force >> gpurun_out/r2e_build.log 2>&1
exit 0
