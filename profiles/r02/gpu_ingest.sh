python profiles/ingest_probe.py 24 4 > gpurun_out/ingest.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ingest_launches.csv python profiles/ingest_probe.py 24 2 > /dev/null 2>&1
cat gpurun_out/ingest.txt
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/ingest_launches.csv")))
hdr = None
out = []
for r in rows:
    if "Kernel Name" in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            out.append((d["ID"], d["Kernel Name"][:60], float(d["Metric Value"])))
for x in out[-80:]:
    print(x)
PY
