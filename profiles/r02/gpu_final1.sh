set -x
mkdir -p gpurun_out/r2s3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python profiles/configs_bench.py --configs 0,1,4,3 --out gpurun_out/r2s3/configs_r02_final2.json > gpurun_out/r2s3/configs_r02_final2.log 2>&1
tail -3 gpurun_out/r2s3/configs_r02_final2.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()"
