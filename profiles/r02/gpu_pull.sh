# in-sweep pull: parity + A/B + bench; ncu source capture of the single kernel; ingest launch list
set -x
mkdir -p gpurun_out/r2s3
timeout 1200 python -m pytest tests/test_gpu_pull.py tests/test_gpu_loop.py tests/test_gpu_engine.py tests/test_gpu_configs.py tests/test_gpu_fullsize.py tests/test_gpu_incremental.py -q -x > gpurun_out/r2s3/pull_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s3/pull_tests.log
tail -3 gpurun_out/r2s3/pull_tests.log
timeout 600 python profiles/pull_ab.py 24 1e-5,1e-4,1e-3 5 > gpurun_out/r2s3/pull_ab24.txt 2>&1
timeout 600 python profiles/pull_ab.py 22 1e-4,1e-3 5 > gpurun_out/r2s3/pull_ab22.txt 2>&1
cat gpurun_out/r2s3/pull_ab24.txt gpurun_out/r2s3/pull_ab22.txt
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2s3/bench_pull.log 2>&1
tail -c 400 gpurun_out/r2s3/bench_pull.log
DYNPR_HOST_LOOP=1 timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:"k_sweep_single" --launch-skip 2 -c 1 -o gpurun_out/r2s3/single_full python profiles/small_probe.py 24 > gpurun_out/r2s3/ncu_single.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv python profiles/ingest_probe.py 24 2 > gpurun_out/r2s3/ingest_launches.csv 2>&1
timeout 600 python profiles/ingest_probe.py 24 4 > gpurun_out/r2s3/ingest_probe.txt 2>&1; cat gpurun_out/r2s3/ingest_probe.txt
