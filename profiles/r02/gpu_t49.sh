# multi-chunk combine folded into the split mseg kernel (A/B via env)
set -x
DYNPR_MSEG_COMBINE=1 DYNPR_SWEEP=split timeout 900 python -m pytest tests/test_gpu_pull.py tests/test_gpu_loop.py tests/test_gpu_engine.py -q -x 2>&1 | tail -2
timeout 1200 python profiles/r02/bisect_ab.py 24 . .:DYNPR_MSEG_COMBINE=1 .:DYNPR_MSEG_COMBINE=1+DYNPR_SINGLE_BPS=2 .:DYNPR_MSEG_COMBINE=1+DYNPR_MSEG_BPS=1
timeout 1200 python profiles/r02/dfp_bisect_ab.py 24:1e-4 . .:DYNPR_MSEG_COMBINE=1 .:DYNPR_MSEG_COMBINE=1+DYNPR_SINGLE_BPS=2 .:DYNPR_MSEG_COMBINE=1+DYNPR_MSEG_BPS=1
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 python -m pytest tests/test_gpu_loop.py -k "all_engines or end_game" -x -q -p no:cacheprovider 2>&1 | grep -E 'ERROR SUMMARY|passed|failed' | tail -2
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 python -m pytest tests/test_gpu_prims.py -k "scan or select" -x -q -p no:cacheprovider 2>&1 | grep -E 'ERROR SUMMARY|passed|failed' | tail -2
