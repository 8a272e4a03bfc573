# copy-through operands loaded with the flags + 4-deep init_ranks
set -x
timeout 900 python -m pytest tests/test_gpu_pull.py tests/test_gpu_engine.py tests/test_gpu_loop.py -q -x 2>&1 | tail -2
timeout 900 python profiles/r02/dfp_bisect_ab.py 24:1e-4,24:1e-5,20:1e-7,20:1e-5,18:1e-4 _ab_head .
timeout 600 python profiles/r02/bisect_ab.py 24 _ab_head .
