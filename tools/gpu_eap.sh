# EAP baseline gate: engine tests (incl. EAP parity) + simulate_decoding smoke of Strategy.eap()
set -x
timeout 900 python -m pytest tests/test_gpu_engine.py -x -q 2>&1 | tail -15 > gpurun_out/pytest_engine.log || exit 3
exit 0
