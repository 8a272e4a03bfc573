set -x
mkdir -p gpurun_out/r2s3
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2s3/t18_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s3/t18_tests.log
tail -3 gpurun_out/r2s3/t18_tests.log
DYNPR_HOST_LOOP=1 timeout 900 ncu --set full --import-source on --clock-control none --kernel-name k_sweep_single --launch-skip 5 -c 1 -o gpurun_out/r2s3/single_flagged_pull python profiles/flagged_once.py 24 > gpurun_out/r2s3/ncu_flagged_pull.log 2>&1
tail -2 gpurun_out/r2s3/ncu_flagged_pull.log
DYNPR_FORCE_TEAM=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2s3/bench_team.log 2>&1; tail -c 1200 gpurun_out/r2s3/bench_team.log
