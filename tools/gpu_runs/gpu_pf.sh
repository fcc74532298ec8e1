# L2 prefetch of the next step's router rows from K3's barrier: tests + all-resident probe + quick bench
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py tests/test_gpu_parity_big.py -x -q 2>&1 | tail -3 > gpurun_out/pf_pytest.log
timeout 300 python tools/k1_probe.py 0:r 0:r > gpurun_out/pf_probe.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-prefill --no-cpu --e2e-steps 1 > gpurun_out/pf_bq.log 2>&1
exit 0
