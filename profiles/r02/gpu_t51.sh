# launch list of the bench command (final code)
set -x
mkdir -p gpurun_out/t51
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/t51/launches_bench_session4.csv python bench.py --steps 2 --warmup 1 > gpurun_out/t51/bench_under_ncu.log 2>&1
echo "exit $?"; wc -l gpurun_out/t51/launches_bench_session4.csv
