set -x
timeout 600 python profiles/hostloop_caps_ab.py 24
