set -x
mkdir -p gpurun_out/r2s3
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2s3/t19_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s3/t19_tests.log
tail -3 gpurun_out/r2s3/t19_tests.log
timeout 600 python profiles/flagged_overhead_probe.py 24
timeout 600 python profiles/r02/bisect_ab.py 24 _ab_head . 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2s3/bench_t19.log 2>&1
python -c "
import json; t=open('gpurun_out/r2s3/bench_t19.log').read(); d=json.loads(t[t.find('{\"metric'):].split(chr(10))[0]); print(d['value'], d['static']['ms_per_solve'], d['dfp'], d['ingest']['ms_per_batch'])"
timeout 600 python profiles/pull_ab.py 20 1e-7,1e-5,1e-4,1e-3 4
