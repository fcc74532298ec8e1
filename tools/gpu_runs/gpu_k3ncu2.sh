# ncu full capture of one standalone K3 launch on the bench mix (source-level stalls)
set -x
K3_ONLY=qwen_bench_mix timeout 600 ncu --set full --import-source on --clock-control none -k regex:ffn_kernel -s 6 -c 1 -o gpurun_out/k3v2_full python tools/profile_kernels.py k3sweep 10 > gpurun_out/k3v2_ncu.log 2>&1
exit 0
