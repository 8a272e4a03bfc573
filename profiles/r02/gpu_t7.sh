set -x
mkdir -p gpurun_out/r2s3
timeout 1200 python -m pytest tests/test_gpu_pull.py tests/test_gpu_loop.py tests/test_gpu_engine.py tests/test_gpu_configs.py tests/test_gpu_acceptance.py -q -x > gpurun_out/r2s3/t7_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s3/t7_tests.log
tail -3 gpurun_out/r2s3/t7_tests.log
timeout 600 python profiles/r02/static_small_ab.py 18 20
timeout 600 python profiles/env_ab.py 24 1e-4 4 DYNPR_LAZY_LISTS=0,1
timeout 600 python profiles/env_ab.py 24 1e-3 4 DYNPR_LAZY_LISTS=0,1
timeout 600 python profiles/env_ab.py 20 1e-4 4 DYNPR_LAZY_LISTS=0,1
timeout 600 python profiles/env_ab.py 20 1e-3 4 DYNPR_LAZY_LISTS=0,1
timeout 600 python profiles/env_ab.py 18 1e-4 4 DYNPR_LAZY_LISTS=0,1
