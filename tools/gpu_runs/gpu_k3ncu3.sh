set -x
K3_SPECS=${K3_SPECS:-int2x4} timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_kernel -s 6 -c 1 -o gpurun_out/k3n3 python tools/profile_kernels.py k3prof 8 > gpurun_out/k3n3.log 2>&1
exit 0
