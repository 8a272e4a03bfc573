# round 2 session 5: final verification after the split-grab change (8 slices, Static and frontier) (suite, smoke, bench, reference arm)
set -x
mkdir -p gpurun_out/r2s5k
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/r2s5k/gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s5k/gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s5k/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r2s5k/smoke.log
timeout 900 python bench.py > gpurun_out/r2s5k/bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/r2s5k/bench_ref.log 2>&1
tail -3 gpurun_out/r2s5k/gputest.log; tail -1 gpurun_out/r2s5k/smoke.log; tail -c 1500 gpurun_out/r2s5k/bench.log; tail -c 600 gpurun_out/r2s5k/bench_ref.log
