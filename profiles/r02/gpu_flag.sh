timeout 600 python profiles/flagged_overhead_probe.py 24
timeout 600 python profiles/dfp_iter_probe.py 24 1e-4 2>&1 | grep -v ' 1.00 m' | sed -n '/^dfp/,$p'
