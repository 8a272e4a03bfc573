# DF-P grid caps, 2-D
set -x
DYNPR_SINGLE_BPS=4 timeout 600 python profiles/env_ab.py 24 1e-4 3 DYNPR_MSEG_BPS=2,1,3
DYNPR_MSEG_BPS=2 timeout 600 python profiles/env_ab.py 24 1e-3 3 DYNPR_SINGLE_BPS=3,4
DYNPR_MSEG_BPS=2 timeout 600 python profiles/env_ab.py 26 1e-4 3 DYNPR_SINGLE_BPS=3,4
DYNPR_MSEG_BPS=2 timeout 600 python profiles/env_ab.py 26 1e-6 3 DYNPR_SINGLE_BPS=3,4
