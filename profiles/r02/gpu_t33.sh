# DF-P grid caps (flagged kernels co-residency)
set -x
timeout 600 python profiles/env_ab.py 24 1e-4 4 DYNPR_SINGLE_BPS=3,2,4,5,0
timeout 600 python profiles/env_ab.py 24 1e-4 4 DYNPR_MSEG_BPS=2,1,3,0
timeout 600 python profiles/env_ab.py 24 1e-5 4 DYNPR_SINGLE_BPS=3,2,4
