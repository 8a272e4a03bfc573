set -x
timeout 1500 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_multi.py tests/test_gpu_loop.py tests/test_gpu_engine.py tests/test_gpu_api.py -q -x --durations=5 > gpurun_out/r2_multi.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2_multi.log
DYNPR_FORCE_TEAM=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_forceteam.log 2>&1
tail -30 gpurun_out/r2_multi.log; tail -c 1500 gpurun_out/r2_forceteam.log
