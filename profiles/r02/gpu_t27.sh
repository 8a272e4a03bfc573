# whole-graph ncu of the device loop (Static + DF-P, RMAT-24)
set -x
mkdir -p gpurun_out/t27
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__cycles_elapsed.avg.per_second,l1tex__m_l1tex2xbar_req_cycles_active.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex.sum,dram__bytes_read.sum,dram__bytes_write.sum
python profiles/r02/graph_once.py 24
timeout 900 ncu --graph-profiling graph --nvtx --nvtx-include "dynpr device loop/" --metrics $M --clock-control none --csv python profiles/r02/graph_once.py 24 > gpurun_out/t27/ncu_graph.csv 2>&1
echo "exit $?"; grep -c k_ gpurun_out/t27/ncu_graph.csv; head -c 3000 gpurun_out/t27/ncu_graph.csv | tail -c 1500
if ! grep -q l1tex__m_l1tex2xbar gpurun_out/t27/ncu_graph.csv; then
  timeout 900 ncu --graph-profiling graph --metrics $M --clock-control none --csv python profiles/r02/graph_once.py 22 > gpurun_out/t27/ncu_graph_all.csv 2>&1
  echo "exit $?"; grep -v '^==PROF' gpurun_out/t27/ncu_graph_all.csv | head -c 2000
fi
