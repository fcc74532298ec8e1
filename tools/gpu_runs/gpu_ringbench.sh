# Bulk-copy ring bandwidth microbenchmark (K3's streaming pattern)
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/bench/bulk_ringbench.cu -o gpurun_out/bulk_ringbench || exit 3
timeout 120 gpurun_out/bulk_ringbench > gpurun_out/ringbench.log 2>&1
exit 0
