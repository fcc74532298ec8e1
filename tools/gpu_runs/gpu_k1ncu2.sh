set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_gate_kernel --launch-skip 100 --launch-count 1 -f -o gpurun_out/k1v3 python tools/k1_probe.py 0:r > gpurun_out/k1v3_ncu.log 2>&1
exit 0
