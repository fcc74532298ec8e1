set -x
timeout 300 python tools/profile_kernels.py allhit 64 > gpurun_out/arc_allhit_side.log 2>&1
FATE_ARC_INLINE=1 timeout 300 python tools/profile_kernels.py allhit 64 > gpurun_out/arc_allhit_inline.log 2>&1
timeout 300 python tools/profile_kernels.py timeline 64 > gpurun_out/arc_tl_side.log 2>&1
FATE_ARC_INLINE=1 timeout 300 python tools/profile_kernels.py timeline 64 > gpurun_out/arc_tl_inline.log 2>&1
FATE_ARC_INLINE=1 timeout 600 python -m pytest tests/test_gpu_engine.py -x -q 2>&1 | tail -3 > gpurun_out/arc_pytest.log
exit 0
