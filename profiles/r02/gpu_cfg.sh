set -x
mkdir -p gpurun_out/r2s3
timeout 1800 python profiles/configs_bench.py --configs 0,1,4 --out gpurun_out/r2s3/configs_r02.json > gpurun_out/r2s3/configs_r02.log 2>&1
tail -40 gpurun_out/r2s3/configs_r02.log
DYNPR_HOST_LOOP=1 timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:"k_sweep_single" --launch-skip 2 -c 1 -o gpurun_out/r2s3/single_full2 python profiles/small_probe.py 24 > gpurun_out/r2s3/ncu_single2.log 2>&1
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
DYNPR_HOST_LOOP=1 timeout 900 ncu --metrics $M --clock-control none --csv --kernel-name regex:"k_sweep_(single|mseg|mfinal)" --launch-skip 3 -c 3 python profiles/small_probe.py 24 > gpurun_out/r2s3/ncu_req_t6.csv 2>&1
python profiles/ncu_request_pipe.py gpurun_out/r2s3/ncu_req_t6.csv
