mkdir -p gpurun_out/r2s3
DYNPR_HOST_LOOP=1 timeout 900 ncu --set full --import-source on --clock-control none --kernel-name k_sweep_single --launch-skip 4 -c 1 -o gpurun_out/r2s3/single_flagged python profiles/flagged_once.py 24 > gpurun_out/r2s3/ncu_flagged.log 2>&1
DYNPR_HOST_LOOP=1 timeout 900 ncu --set full --import-source on --clock-control none --kernel-name k_sweep_single --launch-skip 1 -c 1 -o gpurun_out/r2s3/single_static python profiles/flagged_once.py 24 > gpurun_out/r2s3/ncu_static.log 2>&1
tail -2 gpurun_out/r2s3/ncu_flagged.log
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2s3/t16_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s3/t16_tests.log
tail -3 gpurun_out/r2s3/t16_tests.log
