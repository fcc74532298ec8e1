set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_gate_kernel -s 40 -c 1 -o gpurun_out/k1_full python tools/profile_kernels.py allhit 16 > gpurun_out/ncu_k1.log 2>&1
exit 0
