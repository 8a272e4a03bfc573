# memcheck over the session-4 paths (IF-node push / end game, rows-driven layout, batch touched rows, scan)
mkdir -p gpurun_out/r2s4
for t in tests/test_gpu_graph.py tests/test_gpu_incremental.py "tests/test_gpu_pull.py -k thresholds" "tests/test_gpu_loop.py -k all_engines or end_game" "tests/test_gpu_prims.py -k scan or select"; do
  timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 99 --print-limit 20 python -m pytest $t -x -q -p no:cacheprovider > gpurun_out/r2s4/memcheck.log 2>&1; echo "$t exit $?"; grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/r2s4/memcheck.log | tail -3
done
