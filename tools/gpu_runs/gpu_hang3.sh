# stall fix (cleared message words, head carries n_od): Mixtral sweep x4, then the full GPU suite
set -x
mkdir -p gpurun_out
rm -f gpurun_out/hang3_summary.log
for i in 1 2 3 4; do
  timeout 600 python -m pytest tests/test_gpu_parity_big.py -k mixtral_budget -x -q > gpurun_out/hang3_$i.log 2>&1
  echo "run $i rc=$?" >> gpurun_out/hang3_summary.log
done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/hang3_pytest.log
exit 0
