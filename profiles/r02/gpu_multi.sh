set -x
timeout 1200 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_multi.py -q -x --durations=10 > gpurun_out/r2_multi.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2_multi.log
tail -30 gpurun_out/r2_multi.log
