# ncu evidence for the bench command: K3 full sections (3 launches) + the launch list.
# FATE_PROFILE_SERIAL=1: K3 is enqueued only after its step's transfers landed (ncu serialises launches).
set -x
FATE_PROFILE_SERIAL=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_kernel -s 200 -c 3 -o gpurun_out/k3_bench_full python bench.py --steps 1 --warmup 1 --tokens 16 --no-cpu --e2e-steps 0 --no-prefill > gpurun_out/ncu_bench_full.log 2>&1
FATE_PROFILE_SERIAL=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ffn_kernel|decode_gate|arc_|run_begin|engine_reset|build_xlay" --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --tokens 8 --no-cpu --e2e-steps 0 --no-prefill > gpurun_out/b_ncu.log 2>&1
exit 0
