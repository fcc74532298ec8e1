# full round-end evidence: tests, smoke, bench, Mixtral sweep, ncu (K3, K4, launch list)
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log || exit 3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 900 python tools/profile_kernels.py mixtral 32 > gpurun_out/mixtral.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ffn_kernel -s 40 -c 1 -o gpurun_out/k3_full python tools/profile_kernels.py allhit 16 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k4_tc_kernel -s 6 -c 2 -o gpurun_out/k4_full python tools/profile_kernels.py prefill 512 > gpurun_out/ncu_k4.log 2>&1
FATE_PROFILE_SERIAL=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ffn_kernel|decode_gate|arc_|run_begin|engine_reset|build_xlay" --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --tokens 8 --no-cpu --e2e-steps 0 --no-prefill > gpurun_out/b_ncu.log 2>&1
exit 0
