timeout 300 python profiles/trace_probe.py 18
timeout 300 python profiles/trace_probe.py 20
timeout 300 python profiles/dfp_iter_probe.py 20 1e-7 2>&1 | sed -n '/^dfp/,$p'
