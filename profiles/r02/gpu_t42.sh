# push expansion item size 1024 (.) vs 512 vs 256 edges
set -x
timeout 1500 python profiles/r02/dfp_bisect_ab.py 20:1e-7,20:1e-5,18:1e-4,u20:1e-4,u20:1e-3,24:1e-4,24:1e-6 . _ab_c512 _ab_c256
