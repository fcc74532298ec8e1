set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 300 python tools/profile_kernels.py k3 200 > gpurun_out/k3.log 2>&1
timeout 300 python tools/profile_kernels.py allhit 64 > gpurun_out/allhit.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --tokens 16 --no-cpu --e2e-steps 0 > gpurun_out/b_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_kernel -s 20 -c 1 -o gpurun_out/k3_full python tools/profile_kernels.py k3 40 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/*.log
