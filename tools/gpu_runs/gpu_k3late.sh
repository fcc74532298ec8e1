# K3 late-expert split: numerics + protocol identity + parity, then cold-decode tail and bench
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py tests/test_gpu_parity_big.py tests/test_gpu_prefill.py -x -q 2>&1 | tail -8 > gpurun_out/split_pytest.log
FATE_HOSTPROF=1 timeout 300 python tools/k1_probe.py 0:c 15:c > gpurun_out/split_probe.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-prefill --no-cpu --e2e-steps 1 > gpurun_out/split_bq.log 2>&1
exit 0
