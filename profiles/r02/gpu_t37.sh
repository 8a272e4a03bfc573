# push expansion inside an IF node of the loop graph
set -x
timeout 1200 python -m pytest tests/test_gpu_pull.py tests/test_gpu_engine.py tests/test_gpu_loop.py tests/test_gpu_harness.py tests/test_gpu_configs.py tests/test_gpu_multi.py tests/test_gpu_api.py -q -x 2>&1 | tail -3
timeout 900 python profiles/r02/dfp_bisect_ab.py u20:1e-4,u20:1e-3 _ab_prev .
timeout 300 python profiles/dfp_iter_probe.py 20 1e-7 2>&1 | grep -A8 '^dfp'
