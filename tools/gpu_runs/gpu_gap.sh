# launch hand-off microbenchmark + warp-1 ARC timing in K1 (profiling build)
set -x
mkdir -p gpurun_out
for a in "1 204800 0" "0 204800 0" "1 0 0" "0 0 0" "1 204800 1" "0 204800 1"; do ./tools/bench/gap_bench $a; done > gpurun_out/gap_bench.log 2>&1
FATE_PROF=1 python -m paper_2502_12224_b200.build --force > gpurun_out/gap2_build.log 2>&1
FATE_HOSTPROF=1 timeout 300 python tools/k1_probe.py 0:r 0:c > gpurun_out/gap2_probe.log 2>&1
python -m paper_2502_12224_b200.build --force >> gpurun_out/gap2_build.log 2>&1
exit 0
