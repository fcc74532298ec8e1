# fence-free tagged decode message: full GPU suite, smoke (also serialised), quick bench
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/msg_pytest.log
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/msg_smoke_blocking.log 2>&1; echo "rc=$?" >> gpurun_out/msg_smoke_blocking.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-prefill --no-cpu --e2e-steps 1 > gpurun_out/msg_bq.log 2>&1
exit 0
