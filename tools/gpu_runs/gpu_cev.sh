set -x
timeout 600 python bench.py --steps 4 --no-cpu --e2e-steps 0 --no-regimes --no-prefill > gpurun_out/cev_on.log 2>&1
FATE_NO_COPY_EVENTS=1 timeout 600 python bench.py --steps 4 --no-cpu --e2e-steps 0 --no-regimes --no-prefill > gpurun_out/cev_off.log 2>&1
exit 0
