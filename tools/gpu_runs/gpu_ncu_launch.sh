set -x
FATE_PROFILE_SERIAL=1 timeout 300 python -m pytest tests/test_gpu_engine.py -x -q 2>&1 | tail -5 > gpurun_out/pytest_serial.log
FATE_PROFILE_SERIAL=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ffn_kernel|decode_gate|arc_|run_begin|engine_reset|k4_|prefill_|gate_batch|build_xlay" --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --tokens 8 --no-cpu --e2e-steps 0 > gpurun_out/b_ncu.log 2>&1
exit 0
