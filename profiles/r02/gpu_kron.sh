set -x
mkdir -p gpurun_out/r2s3
timeout 900 python profiles/kron_ingest_probe.py 27 4
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s3/kron_ingest_launches.csv python profiles/kron_ingest_probe.py 27 2 > /dev/null 2>&1
timeout 600 python profiles/dfp_iter_probe.py 24 1e-4 2>&1 | grep -v ' 1.00 m' | head -24
