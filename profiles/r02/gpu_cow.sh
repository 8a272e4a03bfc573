set -x
mkdir -p gpurun_out/r2s3
timeout 2400 python -m pytest tests -q -m gpu -x --durations=5 > gpurun_out/r2s3/t4_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s3/cow_tests.log
tail -12 gpurun_out/r2s3/t4_tests.log
timeout 600 python profiles/ingest_probe.py 24 4 > gpurun_out/r2s3/ingest_probe4.txt 2>&1; cat gpurun_out/r2s3/ingest_probe3.txt
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2s3/bench_t4.log 2>&1
tail -c 1200 gpurun_out/r2s3/bench_t4.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv python profiles/ingest_probe.py 24 2 > gpurun_out/r2s3/ingest_launches4.csv 2>&1
