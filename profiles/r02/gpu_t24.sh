set -x
timeout 1200 python -m pytest tests/test_gpu_prims.py -q -x 2>&1 | tail -4
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 99 python -m pytest tests/test_gpu_prims.py -q -x -k "1025 or 4097 or 262145" -p no:cacheprovider 2>&1 | grep -E 'ERROR SUMMARY|passed|failed' | tail -2
