set -x
timeout 1500 python profiles/r02/bisect_ab.py 18,20 _ab_old _ab_77d67a0 _ab_a6b8ab7 _ab_07adea0 _ab_f833636 _ab_9ec9305 _ab_d4a6c2c .
timeout 600 python profiles/r02/bisect_ab.py 24 _ab_d4a6c2c .
