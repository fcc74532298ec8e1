set -x
nvidia-smi -L
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r2d_pytest.log
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke_blocking.log 2>&1
echo rc=$? >> gpurun_out/r2d_smoke_blocking.log
timeout 600 python bench.py > gpurun_out/r2d_bench.log 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke_ncu.log 2>&1
echo ncu_rc=$? >> gpurun_out/r2d_smoke_ncu.log
exit 0
