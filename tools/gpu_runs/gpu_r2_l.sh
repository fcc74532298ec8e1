set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_kernel -s 200 -c 1 -o gpurun_out/r2l_k3_bench_full python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 0 --no-prefill > gpurun_out/r2l_k3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k4_tc_kernel -s 4 -c 2 -o gpurun_out/r2l_k4_full python tools/profile_kernels.py prefill 512 > gpurun_out/r2l_k4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_gate_kernel -s 200 -c 1 -o gpurun_out/r2l_k1_full python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 0 --no-prefill > gpurun_out/r2l_k1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2l_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 0 --no-prefill --tokens 16 > gpurun_out/r2l_launch.log 2>&1
exit 0
