set -x
for c in 3.0f 2.4f 3.6f 4.2f; do
  FATE_PROF=1 FATE_DEFS="FATE_K3_COST2=$c" python -m paper_2502_12224_b200.build --force > /dev/null 2>&1
  echo "### COST2=$c" >> gpurun_out/k3cost.log
  K3_SPECS=qwen_bench_mix timeout 300 python tools/profile_kernels.py k3prof 20 2>&1 | head -10 >> gpurun_out/k3cost.log
done
python -m paper_2502_12224_b200.build --force > /dev/null 2>&1
exit 0
