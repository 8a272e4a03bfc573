set -x
timeout 900 python -m pytest tests/test_gpu_pull.py tests/test_gpu_engine.py -q -x 2>&1 | tail -2
DYNPR_HEAVY_LANES=2 timeout 600 python -m pytest tests/test_gpu_pull.py -q -x 2>&1 | tail -2
timeout 900 python profiles/r02/bisect_ab.py 16,17,18,19,20 _ab_head .:DYNPR_HEAVY_LANES=1 .:DYNPR_HEAVY_LANES=2
timeout 600 python profiles/r02/dfp_bisect_ab.py 18:1e-4,19:1e-4,18:1e-3 _ab_head .:DYNPR_HEAVY_LANES=1 .:DYNPR_HEAVY_LANES=2
