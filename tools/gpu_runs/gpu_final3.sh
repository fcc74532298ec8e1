# round-end: validation (tests, smoke, bench, reference arm, peer), then the ncu evidence of the bench command
set -x
bash tools/gpu_final2.sh || exit 3
bash tools/gpu_ncu_bench.sh
exit 0
