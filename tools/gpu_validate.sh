# Round-end checks on a B200 box (run through gpurun from the repo root):
# the GPU suite, smoke (also under launch serialisation), the bench line, the
# reference arm, the ncu launch list of smoke, and a 2-rank functional run.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_blocking.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches.csv \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu.log 2>&1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29655 \
  bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 --no-prefill --no-regimes --peer-fetch > gpurun_out/bench_2rank.log 2>&1
exit 0
