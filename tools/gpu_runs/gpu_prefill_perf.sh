set -x
timeout 600 python tools/profile_kernels.py prefill 512 > gpurun_out/prefill_perf.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k4_tc_kernel -s 6 -c 2 -o gpurun_out/k4_full python tools/profile_kernels.py prefill 512 > gpurun_out/ncu_k4.log 2>&1
exit 0
