set -x
timeout 300 python tools/profile_kernels.py allhit 64 > gpurun_out/k1_allhit.log 2>&1
timeout 300 python tools/profile_kernels.py timeline 64 > gpurun_out/k1_timeline.log 2>&1
FATE_PROF=1 python -m paper_2502_12224_b200.build --force > gpurun_out/k1_build.log 2>&1
timeout 300 python tools/profile_kernels.py allhit 64 > gpurun_out/k1_allhit_prof.log 2>&1
python -m paper_2502_12224_b200.build --force >> gpurun_out/k1_build.log 2>&1
exit 0
