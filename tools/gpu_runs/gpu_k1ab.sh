# K1 hand-off change gate: engine parity, then stamps (profiling build) with the
# cooperative and non-cooperative K3 launch
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_parity_big.py -x -q 2>&1 | tail -3 > gpurun_out/ab_pytest.log
FATE_PROF=1 python -m paper_2502_12224_b200.build --force > gpurun_out/ab_build.log 2>&1
timeout 300 python tools/profile_kernels.py allhit 64 2>&1 | grep -v "^ " | tail -3 > gpurun_out/ab_allhit.log
FATE_HOSTPROF=1 timeout 300 python tools/k1_probe.py 0:r 0:c > gpurun_out/ab_probe_coop.log 2>&1
FATE_K3_NONCOOP=1 FATE_HOSTPROF=1 timeout 300 python tools/k1_probe.py 0:r 0:c > gpurun_out/ab_probe_noncoop.log 2>&1
python -m paper_2502_12224_b200.build --force >> gpurun_out/ab_build.log 2>&1
exit 0
