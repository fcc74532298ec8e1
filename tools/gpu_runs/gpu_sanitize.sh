set -x
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 python -m pytest tests/test_gpu_kernels.py -x -q -k "ffn or quant" > gpurun_out/sanitize_kernels.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_kernels.log
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 python -m pytest tests/test_gpu_prefill.py -x -q -k "standalone or multi_tile" > gpurun_out/sanitize_prefill.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_prefill.log
exit 0
