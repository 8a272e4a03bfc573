set -x
mkdir -p gpurun_out/t41
DYNPR_HOST_LOOP=1 timeout 600 ncu --nvtx --nvtx-include "dynpr_dynamic_frontier/" --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv python profiles/dfp_once.py 20 1e-7 > gpurun_out/t41/dfp20_launches.csv 2>&1
python - <<'PY'
import csv, io
f = "gpurun_out/t41/dfp20_launches.csv"
t = open(f).read(); i = t.find('"ID"')
rows = list(csv.reader(io.StringIO(t[i:])))
h = rows[0]; k = h.index("Kernel Name"); v = h.index("Metric Value"); g = h.index("Grid Size")
for r in rows[1:]:
    if len(r) == len(h): print("%-50s %-14s %10s" % (r[k][:50], r[g], r[v]))
PY
