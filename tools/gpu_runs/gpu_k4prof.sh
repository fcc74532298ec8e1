set -x
FATE_PROF=1 python -m paper_2502_12224_b200.build --force > gpurun_out/k4p_build.log 2>&1
timeout 600 python tools/profile_kernels.py k4prof 512 > gpurun_out/k4prof.log 2>&1
python -m paper_2502_12224_b200.build --force >> gpurun_out/k4p_build.log 2>&1
exit 0
