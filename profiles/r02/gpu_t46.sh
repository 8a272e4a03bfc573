# Kron-27 warm ingest breakdown
set -x
mkdir -p gpurun_out/t46
timeout 600 python profiles/kron_ingest_probe.py 27 4
timeout 900 ncu --nvtx --nvtx-include "dynpr_graph_prepare/" --nvtx-include "dynpr_graph_apply_batch_pair/" --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv python profiles/kron_ingest_probe.py 27 2 > gpurun_out/t46/kron_ingest_launches.csv 2>&1
python - <<'PY'
import csv, io, collections
t = open("gpurun_out/t46/kron_ingest_launches.csv").read(); i = t.find('"ID"')
rows = list(csv.reader(io.StringIO(t[i:])))
h = rows[0]; k = h.index("Kernel Name"); v = h.index("Metric Value"); g = h.index("Grid Size")
rows = [r for r in rows[1:] if len(r) == len(h)]
print(len(rows), "launches")
# the last rep's kernels: after the last k_apply... print the last 80 launches
for r in rows[-90:]:
    print("%-60s %-16s %10s" % (r[k][:60], r[g], r[v]))
PY
