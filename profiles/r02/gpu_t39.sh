# loop bookkeeping folded into the latency-mode sweep's last CTA
set -x
timeout 1200 python -m pytest tests/test_gpu_pull.py tests/test_gpu_engine.py tests/test_gpu_loop.py tests/test_gpu_harness.py tests/test_gpu_configs.py tests/test_gpu_api.py -q -x 2>&1 | tail -3
timeout 900 python profiles/r02/bisect_ab.py 16,18,20,22 _ab_prev .
timeout 900 python profiles/r02/dfp_bisect_ab.py 20:1e-7,20:1e-5,18:1e-4,22:1e-4,u20:1e-3 _ab_prev .
