set -x
timeout 1500 python tools/run_b200_experiments.py 64 > gpurun_out/r2h_experiments.log 2>&1
mkdir -p gpurun_out/r02_experiments; cp -r profiles/r02_experiments/* gpurun_out/r02_experiments/ 2>/dev/null
exit 0
