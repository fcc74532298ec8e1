# EAP baseline gate: engine + prefill tests (incl. EAP decode / prefill->decode parity)
set -x
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_prefill.py -x -q 2>&1 | tail -25 > gpurun_out/pytest_engine.log || exit 3
exit 0
