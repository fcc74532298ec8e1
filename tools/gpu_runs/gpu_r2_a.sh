set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2a_pytest.log
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke_blocking.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2a_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke_ncu.log 2>&1
echo ncu_rc=$? >> gpurun_out/r2a_smoke_ncu.log
exit 0
