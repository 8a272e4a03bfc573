set -x
timeout 1500 python profiles/r02/bisect_ab.py 18,20,22 _ab_a6b8ab7 _ab_nofold . .:DYNPR_NO_SELF_FAST=1
timeout 600 python profiles/first_call_probe.py
