# profiling build of K3 (phase stamps), then the per-CTA / per-stage timeline
set -x
FATE_PROF=1 python -m paper_2502_12224_b200.build --force > gpurun_out/k3prof_build.log 2>&1
timeout 300 python tools/profile_kernels.py k3prof 20 > gpurun_out/k3prof.log 2>&1
python -m paper_2502_12224_b200.build --force >> gpurun_out/k3prof_build.log 2>&1
exit 0
