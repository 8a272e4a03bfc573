# DF-P: an iteration that leaves nothing affected accounts the next (empty) one without its sweep
set -x
timeout 1500 python -m pytest tests/test_gpu_pull.py tests/test_gpu_engine.py tests/test_gpu_loop.py tests/test_gpu_configs.py tests/test_gpu_harness.py tests/test_gpu_harness_golden.py tests/test_gpu_api.py tests/test_gpu_acceptance.py tests/test_gpu_compat.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -3
timeout 1500 python profiles/r02/dfp_bisect_ab.py 24:1e-4,24:1e-3,20:1e-7,20:1e-5,u20:1e-4 _ab_prev .
timeout 300 python profiles/dfp_iter_probe.py 24 1e-4 2>&1 | grep -A16 '^dfp'
