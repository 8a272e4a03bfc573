set -x
mkdir -p gpurun_out/r2s3
timeout 1200 python -m pytest tests/test_gpu_pull.py tests/test_gpu_loop.py tests/test_gpu_engine.py tests/test_gpu_configs.py tests/test_gpu_acceptance.py -q -x > gpurun_out/r2s3/fp_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s3/fp_tests.log
tail -2 gpurun_out/r2s3/fp_tests.log
timeout 600 python profiles/pull_ab.py 20 1e-7,1e-6,1e-5,1e-4,1e-3 5 > gpurun_out/r2s3/pull_ab20.txt 2>&1; cat gpurun_out/r2s3/pull_ab20.txt
timeout 600 python profiles/pull_ab.py 18 1e-4,1e-3 5 > gpurun_out/r2s3/pull_ab18.txt 2>&1; cat gpurun_out/r2s3/pull_ab18.txt
for a in "20 1e-4" "20 1e-7"; do timeout 300 python profiles/dfp_iter_probe.py $a; done 2>&1 | grep -v ' 1.00 m' > gpurun_out/r2s3/iter20.txt; cat gpurun_out/r2s3/iter20.txt
