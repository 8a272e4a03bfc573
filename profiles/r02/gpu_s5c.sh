# session 5: sparse frontier sweeps -- parity (new tests + full suite), A/B vs
# the previous build and vs DYNPR_SPARSE=0, per-iteration trace
set -x
mkdir -p gpurun_out/r2s5c
timeout 900 python -m pytest tests/test_gpu_sparse.py -q -x > gpurun_out/r2s5c/sparse_tests.log 2>&1; tail -3 gpurun_out/r2s5c/sparse_tests.log
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2s5c/gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s5c/gputest.log; tail -3 gpurun_out/r2s5c/gputest.log
timeout 1500 python profiles/r02/dfp_bisect_ab.py 20:1e-7,20:1e-6,20:1e-5,18:1e-4,u20:1e-5,u20:1e-4,24:1e-6,24:1e-5,24:1e-4 _ab_prev . .:DYNPR_SPARSE=0 > gpurun_out/r2s5c/dfp_ab.txt 2>&1
timeout 900 python profiles/r02/bisect_ab.py 20,24 _ab_prev . > gpurun_out/r2s5c/static_ab.txt 2>&1
for a in "20 1e-7" "24 1e-6"; do timeout 300 python profiles/dfp_iter_probe.py $a 2>&1 | grep -A12 '^dfp'; done > gpurun_out/r2s5c/iter.txt
cat gpurun_out/r2s5c/dfp_ab.txt gpurun_out/r2s5c/static_ab.txt gpurun_out/r2s5c/iter.txt
