set -x
mkdir -p gpurun_out/t32
DYNPR_HOST_LOOP=1 timeout 600 ncu --nvtx --nvtx-include "dynpr_dynamic_frontier/" --metrics gpu__time_duration.sum --clock-control none --csv python profiles/dfp_once.py 24 1e-4 > gpurun_out/t32/dfp_launches.csv 2>&1
timeout 600 ncu --graph-profiling graph --nvtx --nvtx-include "dynpr_dynamic_frontier/" --metrics gpu__time_duration.sum --clock-control none --csv python profiles/dfp_once.py 24 1e-4 > gpurun_out/t32/dfp_graph_launches.csv 2>&1
python - <<'PY'
import csv, io
for f in ("gpurun_out/t32/dfp_launches.csv", "gpurun_out/t32/dfp_graph_launches.csv"):
    t = open(f).read(); i = t.find('"ID"')
    rows = list(csv.reader(io.StringIO(t[i:])))
    h = rows[0]; k = h.index("Kernel Name"); v = h.index("Metric Value")
    print("==", f, len(rows) - 1)
    for r in rows[1:]:
        if len(r) == len(h): print("%-60s %10s" % (r[k][:60], r[v]))
PY
