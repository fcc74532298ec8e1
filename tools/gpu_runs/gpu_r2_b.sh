set -x
ncu --metrics gpu__time_duration.sum python -c "import os; print({k:v for k,v in os.environ.items() if 'INJ' in k or 'NV_' in k or 'PRELOAD' in k or 'NSIGHT' in k})" > gpurun_out/r2b_ncu_env.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r2b_pytest.log
timeout 300 python tools/profile_kernels.py k3sweep 50 > gpurun_out/r2b_k3sweep.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 1 --no-prefill > gpurun_out/r2b_bench.log 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke_ncu.log 2>&1
echo ncu_rc=$? >> gpurun_out/r2b_smoke_ncu.log
exit 0
