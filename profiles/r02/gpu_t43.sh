# whole-graph ncu: Static vs DF-P instruction / occupancy / request metrics (RMAT-24)
set -x
mkdir -p gpurun_out/t43
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_requests_srcunit_tex.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,sm__cycles_active.avg,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed_op_global_ld.sum,smsp__inst_executed_op_global_st.sum
timeout 900 ncu --graph-profiling graph --nvtx --nvtx-include "dynpr device loop/" --metrics $M --clock-control none --csv python profiles/r02/graph_once.py 24 > gpurun_out/t43/ncu_graph2.csv 2>&1
python - <<'PY'
import csv, io, collections
t = open("gpurun_out/t43/ncu_graph2.csv").read(); i = t.find('"ID"')
rows = list(csv.reader(io.StringIO(t[i:])))
h = rows[0]; ii = h.index("ID"); mi = h.index("Metric Name"); vi = h.index("Metric Value")
per = collections.OrderedDict()
for r in rows[1:]:
    if len(r) == len(h): per.setdefault(r[ii], {})[r[mi]] = r[vi]
for k, m in per.items():
    print("== graph", k)
    for n, v in m.items(): print("  %-75s %s" % (n, v))
PY
