set -x
mkdir -p gpurun_out/r2s3
timeout 2400 python profiles/configs_bench.py --configs 0,1,4,3 --out gpurun_out/r2s3/configs_r02_final.json > gpurun_out/r2s3/configs_r02_final.log 2>&1
tail -5 gpurun_out/r2s3/configs_r02_final.log
