set -x
mkdir -p gpurun_out/r2s3
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2s3/t6_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s3/t6_tests.log
tail -3 gpurun_out/r2s3/t6_tests.log
timeout 600 python profiles/env_ab.py 24 1e-4 4 DYNPR_INIT_PULL_DIV=0,4,8,16,64,1000000000
timeout 600 python profiles/env_ab.py 24 1e-5 4 DYNPR_INIT_PULL_DIV=0,8,64,1000000000
timeout 600 python profiles/env_ab.py 24 1e-3 4 DYNPR_INIT_PULL_DIV=0,8,64,1000000000
timeout 600 python profiles/env_ab.py 20 1e-4 4 DYNPR_INIT_PULL_DIV=0,8,64,1000000000
timeout 600 python profiles/env_ab.py 20 1e-6 4 DYNPR_INIT_PULL_DIV=0,8,64,1000000000
