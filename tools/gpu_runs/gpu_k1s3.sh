set -x
mkdir -p gpurun_out
FATE_PROF=1 python -m paper_2502_12224_b200.build --force > gpurun_out/s3_build.log 2>&1
FATE_HOSTPROF=1 timeout 300 python tools/k1_probe.py 0:r 0:c > gpurun_out/s3_probe.log 2>&1
python -m paper_2502_12224_b200.build --force >> gpurun_out/s3_build.log 2>&1
exit 0
