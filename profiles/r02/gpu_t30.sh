set -x
timeout 600 python profiles/r02/dfp_first_probe.py 24 6
