set -x
mkdir -p gpurun_out/r2s3
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2s3/t5_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s3/t5_tests.log
tail -3 gpurun_out/r2s3/t5_tests.log
timeout 600 python profiles/ingest_probe.py 24 4 > gpurun_out/r2s3/ingest_probe5.txt 2>&1; cat gpurun_out/r2s3/ingest_probe5.txt
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2s3/bench_t5.log 2>&1
tail -c 1500 gpurun_out/r2s3/bench_t5.log
timeout 600 python profiles/dfp_iter_probe.py 24 1e-4 2>&1 | grep -v ' 1.00 m' | head -30
