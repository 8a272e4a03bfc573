set -x
timeout 1200 python -m pytest tests/test_gpu_loop.py tests/test_gpu_engine.py tests/test_gpu_pull.py -q -x 2>&1 | tail -2
timeout 900 python profiles/r02/bisect_ab.py 24,20,18 _ab_head . _ab_head .
timeout 900 python profiles/r02/dfp_bisect_ab.py 24:1e-4,20:1e-4 _ab_head .
