# timing experiment: K1 event without warp 1's ARC list write-back (results wrong by design)
set -x
mkdir -p gpurun_out
timeout 300 python tools/k1_probe.py 0:r 0:r > gpurun_out/as_base.log 2>&1
FATE_DEFS=FATE_EXP_NOARCSTORE python -m paper_2502_12224_b200.build --force > gpurun_out/as_build.log 2>&1
timeout 300 python tools/k1_probe.py 0:r 0:r > gpurun_out/as_nostore.log 2>&1
python -m paper_2502_12224_b200.build --force >> gpurun_out/as_build.log 2>&1
exit 0
