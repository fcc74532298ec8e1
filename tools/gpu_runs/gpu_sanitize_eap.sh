# memcheck over this session's new device code: EAP decode / prefill (tiny), multi-producer K3
set -x
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 python -m pytest tests/test_gpu_engine.py tests/test_gpu_prefill.py -x -q -k "eap and tiny" > gpurun_out/sanitize_eap.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_eap.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 python -m pytest tests/test_gpu_kernels.py -x -q -k "ffn" > gpurun_out/sanitize_kernels.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_kernels.log
exit 0
