mkdir -p gpurun_out/r2s3
for t in tests/test_gpu_graph.py tests/test_gpu_incremental.py "tests/test_gpu_pull.py -k thresholds" "tests/test_gpu_loop.py -k all_engines"; do
  timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 python -m pytest $t -x -q -p no:cacheprovider > gpurun_out/r2s3/memcheck.log 2>&1; echo "$t exit $?"; grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/r2s3/memcheck.log | tail -3
done
