# round-end check list on the stall-fixed HEAD + bench launch list
set -x
mkdir -p gpurun_out
bash tools/gpu_validate.sh
FATE_PROFILE_SERIAL=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ffn_kernel|decode_gate|arc_|run_begin|engine_reset|build_xlay" --csv --log-file gpurun_out/launches_v4.csv python bench.py --steps 1 --warmup 1 --tokens 8 --no-cpu --e2e-steps 0 --no-prefill --no-regimes > gpurun_out/b_ncu_v4.log 2>&1
exit 0
