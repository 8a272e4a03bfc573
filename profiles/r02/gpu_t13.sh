set -x
mkdir -p gpurun_out/r2s3
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2s3/t13_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s3/t13_tests.log
tail -3 gpurun_out/r2s3/t13_tests.log
timeout 600 python profiles/env_ab.py 24 1e-4 4 DYNPR_MSEG_BPS=0,2
timeout 600 python profiles/env_ab.py 24 1e-3 3 DYNPR_MSEG_BPS=0,2
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2s3/bench_t13.log 2>&1
tail -c 2000 gpurun_out/r2s3/bench_t13.log
