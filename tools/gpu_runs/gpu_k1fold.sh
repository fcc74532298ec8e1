# ARC update folded into K1: engine/cache parity, then the hand-off diagnostics
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_cache_protocol.py tests/test_gpu_parity_big.py tests/test_gpu_prefill.py -x -q 2>&1 | tail -15 > gpurun_out/fold_pytest.log
FATE_PROF=1 python -m paper_2502_12224_b200.build --force > gpurun_out/fold_build.log 2>&1
FATE_HOSTPROF=1 timeout 300 python tools/k1_probe.py 0:r 0:c > gpurun_out/fold_probe.log 2>&1
python -m paper_2502_12224_b200.build --force >> gpurun_out/fold_build.log 2>&1
timeout 300 python tools/k1_probe.py 0:r 0:c 15:c > gpurun_out/fold_probe_prod.log 2>&1
exit 0
