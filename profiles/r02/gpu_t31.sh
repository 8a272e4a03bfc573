set -x
timeout 300 python profiles/dfp_iter_probe.py 24 1e-4 2>&1 | grep -v '^  it  [3-5][0-9] \|^  it  [6-9] \|^  it  [1-2][0-9] ' 
