set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2m_pytest.log
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2m_smoke_blocking.log 2>&1
echo rc=$? >> gpurun_out/r2m_smoke_blocking.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2m_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2m_smoke_ncu.log 2>&1
echo ncu_rc=$? >> gpurun_out/r2m_smoke_ncu.log
timeout 900 python bench.py --impl reference > gpurun_out/r2m_ref.log 2>&1
echo rc=$? >> gpurun_out/r2m_ref.log
exit 0
