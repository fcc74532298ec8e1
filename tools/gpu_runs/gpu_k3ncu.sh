set -x
K3_ONLY=int4x4 timeout 300 ncu --set full --clock-control none --import-source on -k regex:ffn_kernel -s 30 -c 1 -o gpurun_out/k3_int4 python tools/profile_kernels.py k3sweep 20 > gpurun_out/ncu_int4.log 2>&1
K3_ONLY=bf16_shared timeout 300 ncu --set full --clock-control none --import-source on -k regex:ffn_kernel -s 30 -c 1 -o gpurun_out/k3_bf16 python tools/profile_kernels.py k3sweep 20 > gpurun_out/ncu_bf16.log 2>&1
exit 0
