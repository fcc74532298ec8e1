# K1 phase stamps on the current kernels (profiling build), all-resident and cold
set -x
mkdir -p gpurun_out
FATE_PROF=1 python -m paper_2502_12224_b200.build --force > gpurun_out/k1s_build.log 2>&1
timeout 300 python tools/profile_kernels.py allhit 64 > gpurun_out/k1s_allhit.log 2>&1
FATE_HOSTPROF=1 timeout 300 python tools/k1_probe.py 0:r 0:c > gpurun_out/k1s_probe.log 2>&1
python -m paper_2502_12224_b200.build --force >> gpurun_out/k1s_build.log 2>&1
exit 0
