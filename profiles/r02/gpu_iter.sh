set -x
mkdir -p gpurun_out/r2s3
for a in "24 1e-4" "24 1e-5" "20 1e-7" "20 1e-4" "20 1e-4 split"; do timeout 300 python profiles/dfp_iter_probe.py $a; done > gpurun_out/r2s3/iter.txt 2>&1
cat gpurun_out/r2s3/iter.txt | grep -v '^  it' 
DYNPR_HOST_LOOP=1 timeout 600 ncu --nvtx --nvtx-include "dynpr_dynamic_frontier/" --metrics gpu__time_duration.sum --clock-control none --csv python profiles/dfp_once.py 20 1e-7 > gpurun_out/r2s3/dfp20_launches.csv 2>&1
DYNPR_HOST_LOOP=1 timeout 600 ncu --nvtx --nvtx-include "dynpr_dynamic_frontier/" --metrics gpu__time_duration.sum --clock-control none --csv python profiles/dfp_once.py 24 1e-4 > gpurun_out/r2s3/dfp24_launches.csv 2>&1
tail -3 gpurun_out/r2s3/dfp20_launches.csv
