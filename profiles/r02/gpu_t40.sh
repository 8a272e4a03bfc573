# batched push expansion (low: 8 targets per round; high: depth 4 vs 8)
set -x
timeout 900 python -m pytest tests/test_gpu_pull.py tests/test_gpu_engine.py tests/test_gpu_rank.py -q -x 2>&1 | tail -2
timeout 1200 python profiles/r02/dfp_bisect_ab.py 20:1e-7,20:1e-5,18:1e-4,u20:1e-4,u20:1e-3,24:1e-4,24:1e-6 _ab_prev . _ab_h8
timeout 300 python profiles/dfp_iter_probe.py 20 1e-7 2>&1 | grep -A8 '^dfp'
