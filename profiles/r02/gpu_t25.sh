set -x
timeout 1200 python -m pytest tests/test_gpu_loop.py tests/test_gpu_engine.py tests/test_gpu_pull.py -q -x 2>&1 | tail -2
timeout 900 python profiles/r02/bisect_ab.py 18,20,22 _ab_head _ab_g1 . _ab_g4
timeout 900 python profiles/r02/dfp_bisect_ab.py 20:1e-4,18:1e-4 _ab_head _ab_g1 . _ab_g4
