set -x
mkdir -p gpurun_out/r2s3
timeout 1200 python -m pytest tests/test_gpu_pull.py tests/test_gpu_loop.py tests/test_gpu_engine.py tests/test_gpu_incremental.py -q -x > gpurun_out/r2s3/t10_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s3/t10_tests.log
tail -2 gpurun_out/r2s3/t10_tests.log
timeout 900 python profiles/r02/bisect_ab.py 24 _ab_d4a6c2c . _ab_d4a6c2c .
timeout 900 python profiles/grid_ab.py 24 -:-,4:2,5:2,4:3,3:3,6:2,3:4,2:5
timeout 600 python profiles/grid_ab.py 22 -:-,4:2,4:3,3:3
for a in "u20 1e-3" "u20 1e-4"; do timeout 300 python profiles/dfp_iter_probe.py $a; done 2>&1 | grep -v ' 1.00 m' | head -60
