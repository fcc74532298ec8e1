set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log || exit 3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python tools/profile_kernels.py timeline 32 > gpurun_out/timeline.log 2>&1
timeout 300 python tools/profile_kernels.py allhit 64 > gpurun_out/allhit.log 2>&1
exit 0
