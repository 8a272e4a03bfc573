# single-kernel occupancy fix (smem 1 KB -> 256 B per block) + DF-P probes
set -x
mkdir -p gpurun_out/r2s3
timeout 1200 python -m pytest tests/test_gpu_pull.py tests/test_gpu_loop.py tests/test_gpu_engine.py tests/test_gpu_rank.py tests/test_gpu_multi.py -q -x > gpurun_out/r2s3/occ_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s3/occ_tests.log
tail -2 gpurun_out/r2s3/occ_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2s3/bench_occ.log 2>&1
tail -c 300 gpurun_out/r2s3/bench_occ.log
timeout 600 python profiles/dfp_iter_probe.py 24 1e-4 > gpurun_out/r2s3/iter24.txt 2>&1; cat gpurun_out/r2s3/iter24.txt
timeout 600 python profiles/dfp_fixed_probe.py 20 > gpurun_out/r2s3/fixed20.txt 2>&1; cat gpurun_out/r2s3/fixed20.txt
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
DYNPR_HOST_LOOP=1 timeout 900 ncu --metrics $M --clock-control none --csv --kernel-name regex:"k_sweep_(single|mseg|mfinal)" --launch-skip 3 -c 3 python profiles/small_probe.py 24 > gpurun_out/r2s3/ncu_req_occ.csv 2>&1
python profiles/ncu_request_pipe.py gpurun_out/r2s3/ncu_req_occ.csv
