# session 5: k_sweep_mfinal register cap A/B (baseline 63-64 regs for the frontier
# instantiations / 48 with spills / 56 = working tree), DF-P set-up launch list
set -x
mkdir -p gpurun_out/r2s5b
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_loop.py tests/test_gpu_pull.py -q -x 2>&1 | tail -2
timeout 1500 python profiles/r02/dfp_bisect_ab.py 24:1e-4,24:1e-6,20:1e-7,20:1e-4,u20:1e-4 _ab_prev . _ab_mf48 > gpurun_out/r2s5b/dfp_ab.txt 2>&1
timeout 900 python profiles/r02/bisect_ab.py 24,20 _ab_prev . _ab_mf48 > gpurun_out/r2s5b/static_ab.txt 2>&1
timeout 300 python profiles/dfp_iter_probe.py 20 1e-7 2>&1 | grep -A8 '^dfp' > gpurun_out/r2s5b/iter20.txt
DYNPR_HOST_LOOP=1 timeout 600 ncu --nvtx --nvtx-include "dynpr_dynamic_frontier/" --metrics gpu__time_duration.sum --clock-control none --csv python profiles/dfp_once.py 20 1e-7 > gpurun_out/r2s5b/dfp20_launches.csv 2>&1
cat gpurun_out/r2s5b/dfp_ab.txt gpurun_out/r2s5b/static_ab.txt gpurun_out/r2s5b/iter20.txt
