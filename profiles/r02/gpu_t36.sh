set -x
timeout 300 python profiles/dfp_iter_probe.py 20 1e-7 2>&1 | grep -v '^  it  [0-9]* .*processed   1048576 '
timeout 300 python profiles/dfp_iter_probe.py 20 1e-5 2>&1 | grep -v '^  it  [0-9]* .*processed   1048576 '
timeout 300 python profiles/dfp_iter_probe.py 24 1e-5 2>&1 | grep -v '^  it  [0-9]* .*processed  16777216 '
