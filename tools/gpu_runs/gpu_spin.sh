# host poll loop without a driver call per spin: engine tests + quick bench
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_parity_big.py -x -q 2>&1 | tail -3 > gpurun_out/sp_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-prefill --no-cpu --e2e-steps 1 > gpurun_out/sp_bq.log 2>&1
exit 0
