# A/B of K3 producer-warp count: numerics gate, allhit engine, Qwen-mix sweep, short bench
set -x
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k ffn 2>&1 | tail -3 > gpurun_out/pytest_k3.log || exit 3
for np in 1 2 4; do
  FATE_K3_PRODUCERS=$np timeout 300 python tools/profile_kernels.py allhit 64 > gpurun_out/allhit_p$np.log 2>&1
  FATE_K3_PRODUCERS=$np K3_ONLY=qwen_mix_int4 timeout 300 python tools/profile_kernels.py k3sweep 40 > gpurun_out/mix_p$np.log 2>&1
  FATE_K3_PRODUCERS=$np K3_ONLY=qwen_mix_int2 timeout 300 python tools/profile_kernels.py k3sweep 40 >> gpurun_out/mix_p$np.log 2>&1
done
for np in 1 4; do
  FATE_K3_PRODUCERS=$np timeout 600 python bench.py --steps 3 --warmup 3 --no-prefill --no-cpu --e2e-steps 0 > gpurun_out/bench_p$np.log 2>&1
done
exit 0
