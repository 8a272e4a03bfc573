# round 2 (session 3): HEAD verification + request-pipe ncu evidence
set -x
mkdir -p gpurun_out/r2s3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/r2s3/gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s3/gputest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r2s3/smoke.log
timeout 900 python bench.py > gpurun_out/r2s3/bench.log 2>&1
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__cycles_elapsed.avg.per_second,l1tex__m_l1tex2xbar_req_cycles_active.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__m_l1tex2xbar_req_cycles_stalled.sum,l1tex__m_l1tex2xbar_throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_sectors.sum,l1tex__m_xbar2l1tex_throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_miss.sum,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__lsuin_requests.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_lgds_cmd_read.sum
DYNPR_HOST_LOOP=1 timeout 900 ncu --metrics $M --clock-control none --csv --kernel-name regex:"k_sweep_(single|mseg|mfinal)" --launch-skip 3 -c 6 python profiles/small_probe.py 24 > gpurun_out/r2s3/ncu_req_sweep.csv 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb3 profiles/microbench_gather3.cu && /tmp/mb3 > gpurun_out/r2s3/mb3.txt 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --kernel-name k_g8_sms -c 10 /tmp/mb3 > gpurun_out/r2s3/ncu_req_mb3.csv 2>&1
tail -3 gpurun_out/r2s3/gputest.log; tail -1 gpurun_out/r2s3/smoke.log; tail -c 600 gpurun_out/r2s3/bench.log
