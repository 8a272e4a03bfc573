set -x
mkdir -p gpurun_out/r2s3
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2s3/t8_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s3/t8_tests.log
tail -3 gpurun_out/r2s3/t8_tests.log
timeout 1500 python profiles/r02/bisect_ab.py 18,20,22 _ab_a6b8ab7 _ab_nofold .
timeout 600 python profiles/pull_ab.py 20 1e-7,1e-5,1e-4,1e-3 4
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2s3/bench_t8.log 2>&1
tail -c 1500 gpurun_out/r2s3/bench_t8.log
