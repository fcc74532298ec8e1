# round-2 (session 4) evidence: the round-end check list + the bench launch list and a K1 capture
set -x
mkdir -p gpurun_out
bash tools/gpu_validate.sh
FATE_PROFILE_SERIAL=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ffn_kernel|decode_gate|arc_|run_begin|engine_reset|build_xlay" --csv --log-file gpurun_out/launches_v3.csv python bench.py --steps 1 --warmup 1 --tokens 8 --no-cpu --e2e-steps 0 --no-prefill --no-regimes > gpurun_out/b_ncu_v3.log 2>&1
FATE_PROFILE_SERIAL=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_gate -s 100 -c 1 -f -o gpurun_out/k1_bench_v3 python bench.py --steps 1 --warmup 1 --tokens 8 --no-cpu --e2e-steps 0 --no-prefill --no-regimes > gpurun_out/k1_ncu_v3.log 2>&1
exit 0
