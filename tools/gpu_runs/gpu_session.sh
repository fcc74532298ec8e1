# one gpurun session: gate on K3 numerics + engine parity, then timings, bench, ncu (outputs in gpurun_out/)
set -x
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k ffn 2>&1 | tail -15 > gpurun_out/pytest_k3.log || exit 3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log || exit 4
FATE_PROFILE_SERIAL=1 timeout 300 python -m pytest tests/test_gpu_engine.py -x -q 2>&1 | tail -5 > gpurun_out/pytest_serial.log
timeout 300 python tools/profile_kernels.py allhit 64 > gpurun_out/allhit.log 2>&1 || exit 5
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1 || exit 6
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ffn_kernel -s 40 -c 1 -o gpurun_out/k3_full python tools/profile_kernels.py allhit 16 > gpurun_out/ncu_full.log 2>&1
FATE_PROFILE_SERIAL=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ffn_kernel|decode_gate|arc_|run_begin|engine_reset|k4_|prefill_|gate_batch" --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --tokens 8 --no-cpu --e2e-steps 0 --no-prefill > gpurun_out/b_ncu.log 2>&1
exit 0
