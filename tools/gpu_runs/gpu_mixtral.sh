# Mixtral-8x7B-shape decode budget sweep (BASELINE configs[3])
set -x
timeout 900 python tools/profile_kernels.py mixtral 32 > gpurun_out/mixtral.log 2>&1
exit 0
