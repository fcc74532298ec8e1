set -x
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_dense.py tests/test_channel.py -x -q > gpurun_out/san_dense.log 2>&1
echo rc=$? >> gpurun_out/san_dense.log
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_engine_dense.py tests/test_gpu_cache_protocol.py -x -q > gpurun_out/san_engine.log 2>&1
echo rc=$? >> gpurun_out/san_engine.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_dense.py -x -q > gpurun_out/san_race.log 2>&1
echo rc=$? >> gpurun_out/san_race.log
exit 0
