set -x
mkdir -p gpurun_out/r2s3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_loop.py tests/test_gpu_pull.py tests/test_gpu_multi.py -q -x 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r2s3/bench_final.log 2>&1
tail -c 3000 gpurun_out/r2s3/bench_final.log
timeout 900 python bench.py --impl reference > gpurun_out/r2s3/bench_ref.log 2>&1
tail -c 1500 gpurun_out/r2s3/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r2s3/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2s3/ncu_bench.log 2>&1
DYNPR_HOST_LOOP=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum --clock-control none --csv --kernel-name regex:"k_sweep_(single|mseg|mfinal)" --launch-skip 3 -c 3 python profiles/small_probe.py 24 > gpurun_out/r2s3/ncu_dram_final.csv 2>&1
python profiles/ncu_request_pipe.py gpurun_out/r2s3/ncu_dram_final.csv
