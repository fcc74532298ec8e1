# K3 numerics gate, per-format sweep (traced), allhit engine profile
set -x
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k ffn 2>&1 | tail -5 > gpurun_out/pytest_k3.log || exit 3
timeout 300 python tools/profile_kernels.py k3sweep 40 > gpurun_out/k3sweep.log 2>&1
timeout 300 python tools/profile_kernels.py allhit 64 > gpurun_out/allhit.log 2>&1
exit 0
