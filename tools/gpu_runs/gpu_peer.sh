set -x
timeout 600 python -m pytest tests/test_gpu_engine.py -x -q -k sharded 2>&1 | tail -40 > gpurun_out/pytest_peer.log || exit 3
#timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu --no-prefill --e2e-steps 0 --peer-fetch > gpurun_out/bench_peer.log 2>&1
exit 0
