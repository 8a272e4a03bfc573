set -x
timeout 600 python profiles/hostloop_caps_ab.py 24
timeout 600 python profiles/hostloop_caps_ab.py 22
