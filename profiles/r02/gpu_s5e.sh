# session 5: Static split single-slice kernel -- next slice's in-degrees loaded one slice
# ahead, 64-register budget for the Static instantiation (A/B vs the previous build)
set -x
mkdir -p gpurun_out/r2s5e
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_loop.py tests/test_gpu_rank.py tests/test_gpu_configs.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
timeout 1500 python profiles/r02/bisect_ab.py 22,24,25,26 _ab_prev . > gpurun_out/r2s5e/static_ab.txt 2>&1
timeout 600 python profiles/r02/dfp_bisect_ab.py 24:1e-4 _ab_prev . > gpurun_out/r2s5e/dfp_ab.txt 2>&1
cat gpurun_out/r2s5e/static_ab.txt gpurun_out/r2s5e/dfp_ab.txt
