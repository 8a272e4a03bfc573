timeout 1500 python -m pytest tests/test_gpu_incremental.py tests/test_gpu_multi.py tests/test_gpu_loop.py tests/test_gpu_engine.py tests/test_gpu_graph.py tests/test_gpu_rank.py tests/test_gpu_harness.py -q -x --durations=5 > gpurun_out/r2_inc.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2_inc.log
tail -40 gpurun_out/r2_inc.log
python profiles/ingest_probe.py 24 4
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_inc.log 2>&1
tail -c 2500 gpurun_out/r2_bench_inc.log
