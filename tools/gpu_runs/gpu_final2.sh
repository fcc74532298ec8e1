# round-end validation: GPU suite, smoke, default bench, reference arm, peer-fetch bench
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log || exit 3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 1 --no-prefill --no-cpu --e2e-steps 0 --peer-fetch > gpurun_out/bench_peer.log 2>&1
exit 0
