set -x
mkdir -p gpurun_out/r2s3
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2s3/t9_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s3/t9_tests.log
tail -3 gpurun_out/r2s3/t9_tests.log
timeout 900 python profiles/r02/bisect_ab.py 24 _ab_d4a6c2c . _ab_d4a6c2c .
timeout 600 python profiles/first_call_probe.py
timeout 600 python profiles/dfp_fixed_probe.py 20 1e-7,1e-5,1e-3 4
