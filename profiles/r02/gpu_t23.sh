set -x
timeout 1200 python -m pytest tests/test_gpu_loop.py tests/test_gpu_engine.py tests/test_gpu_configs.py -q -x 2>&1 | tail -2
timeout 900 python profiles/r02/bisect_ab.py 24,22 _ab_head _ab_nopair . _ab_head _ab_nopair .
