set -x
timeout 900 python bench.py --steps 3 --warmup 3 --no-prefill > gpurun_out/bench_quick.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
exit 0
