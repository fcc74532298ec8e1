# quick bench A/B: K1 with and without PDL (decode headline + regimes, no prefill / CPU legs)
set -x
mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 3 --no-prefill --no-cpu --e2e-steps 1 > gpurun_out/bq_pdl.log 2>&1
FATE_K1_NOPDL=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-prefill --no-cpu --e2e-steps 1 > gpurun_out/bq_nopdl.log 2>&1
exit 0
