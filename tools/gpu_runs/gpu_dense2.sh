set -x
timeout 600 python -m pytest tests/test_gpu_dense.py tests/test_gpu_engine_dense.py -x -q 2>&1 | tail -20 > gpurun_out/dense2_pytest.log
python tools/dense_probe.py > gpurun_out/dense2_probe.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:gemv|rope|attn" -c 8 --csv --log-file gpurun_out/dense2_launches.csv python tools/dense_probe.py > /dev/null 2>&1
exit 0
