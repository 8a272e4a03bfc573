# session 5: push-expansion grid size (CTAs/SM) A/B on DF-P, tiny-batch parity tests
set -x
mkdir -p gpurun_out/r2s5d
timeout 900 python -m pytest tests/test_gpu_tiny_batches.py -q -x 2>&1 | tail -2
timeout 2000 python profiles/r02/dfp_bisect_ab.py 20:1e-7,20:1e-5,20:1e-3,18:1e-4,u20:1e-5,u20:1e-3,24:1e-6,24:1e-4 .:DYNPR_EXPAND_BPS=16 .:DYNPR_EXPAND_BPS=8 .:DYNPR_EXPAND_BPS=4 .:DYNPR_EXPAND_BPS=2 > gpurun_out/r2s5d/expand_bps_ab.txt 2>&1
cat gpurun_out/r2s5d/expand_bps_ab.txt
