set -x
timeout 300 python tools/profile_kernels.py allhit 64 > gpurun_out/allhit.log 2>&1
exit 0
