set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -q -m gpu -x --durations=25 > gpurun_out/r2_gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2_gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2_bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/r2_bench_ref.log 2>&1
tail -3 gpurun_out/r2_gputest.log; tail -2 gpurun_out/r2_bench.log; tail -2 gpurun_out/r2_bench_ref.log
