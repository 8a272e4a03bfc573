# BASELINE configs with the session-4 code
set -x
mkdir -p gpurun_out/r2s4
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python profiles/configs_bench.py --configs 0,1,4,3 --out gpurun_out/r2s4/configs_r02_s4.json > gpurun_out/r2s4/configs_r02_s4.log 2>&1
tail -40 gpurun_out/r2s4/configs_r02_s4.log
