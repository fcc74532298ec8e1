set -x
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_prefill.py -x -q 2>&1 | tail -30 > gpurun_out/r2i_pytest.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --e2e-steps 1 --no-prefill --peer-fetch > gpurun_out/r2i_bench2.log 2>&1
echo rc=$? >> gpurun_out/r2i_bench2.log
ls /dev/shm >> gpurun_out/r2i_bench2.log
exit 0
