# relabel tiebreak by out-degree (locality experiment)
set -x
DYNPR_RELABEL_TIE=out timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_pull.py -q -x 2>&1 | tail -2
timeout 900 python profiles/r02/bisect_ab.py 20,22,24 . .:DYNPR_RELABEL_TIE=out
timeout 600 python profiles/r02/dfp_bisect_ab.py 24:1e-4,22:1e-4 . .:DYNPR_RELABEL_TIE=out
