set -x
mkdir -p gpurun_out/r2s3
timeout 2400 python -m pytest tests -q -m gpu -x --durations=10 > gpurun_out/r2s3/ing_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s3/ing_tests.log
tail -25 gpurun_out/r2s3/ing_tests.log
timeout 600 python profiles/ingest_probe.py 24 4 > gpurun_out/r2s3/ingest_probe2.txt 2>&1; cat gpurun_out/r2s3/ingest_probe2.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv python profiles/ingest_probe.py 24 2 > gpurun_out/r2s3/ingest_launches2.csv 2>&1
