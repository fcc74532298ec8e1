set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_parity_big.py -x -q 2>&1 | tail -3 > gpurun_out/s4_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-prefill --no-cpu --e2e-steps 1 > gpurun_out/s4_bq.log 2>&1
FATE_PROF=1 python -m paper_2502_12224_b200.build --force > gpurun_out/s4_build.log 2>&1
FATE_HOSTPROF=1 timeout 300 python tools/k1_probe.py 0:r 0:c > gpurun_out/s4_probe.log 2>&1
python -m paper_2502_12224_b200.build --force >> gpurun_out/s4_build.log 2>&1
exit 0
