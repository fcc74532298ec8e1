# K1 v2 (in-K1 ARC update from smem, PDL behind K3): parity, diagnostics, probe
set -x
mkdir -p gpurun_out
for a in "1 204800 0 0" "1 204800 0 2" "1 204800 1 0"; do ./tools/bench/gap_bench $a; done > gpurun_out/v2_gap_bench.log 2>&1
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_cache_protocol.py tests/test_gpu_parity_big.py tests/test_gpu_prefill.py tests/test_gpu_engine_dense.py -x -q 2>&1 | tail -15 > gpurun_out/v2_pytest.log
timeout 300 python tools/k1_probe.py 0:r 0:c 15:c > gpurun_out/v2_probe_prod.log 2>&1
FATE_K1_NOPDL=1 timeout 300 python tools/k1_probe.py 0:r 0:c > gpurun_out/v2_probe_nopdl.log 2>&1
FATE_PROF=1 python -m paper_2502_12224_b200.build --force > gpurun_out/v2_build.log 2>&1
FATE_HOSTPROF=1 timeout 300 python tools/k1_probe.py 0:r 0:c > gpurun_out/v2_probe.log 2>&1
python -m paper_2502_12224_b200.build --force >> gpurun_out/v2_build.log 2>&1
exit 0
