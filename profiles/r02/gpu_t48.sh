# derived layout: slice / chunk passes driven by the touched rows
set -x
timeout 1500 python -m pytest tests/test_gpu_incremental.py tests/test_gpu_graph.py tests/test_gpu_engine.py tests/test_gpu_pull.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -3
for d in _ab_prev .; do echo "== $d"; DYNPR_PKG_ROOT=$PWD/$d timeout 300 python profiles/ingest_probe.py 24 4 2>&1 | tail -3; done
for d in _ab_prev .; do echo "== $d"; DYNPR_PKG_ROOT=$PWD/$d timeout 600 python profiles/kron_ingest_probe.py 27 4 2>&1 | tail -3; done
