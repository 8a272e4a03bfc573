set -x
timeout 900 python profiles/grid_ab.py 24 -:-,3:4,2:4,3:5,4:4,2:3,1:4,3:-,-:4,2:2
for a in "24 1e-4" "24 1e-3" "24 1e-5" "20 1e-7" "20 1e-5" "20 1e-4" "20 1e-3" "u20 1e-3" "u20 1e-4" "18 1e-4"; do timeout 300 python profiles/env_ab.py $a 4 DYNPR_PUSH_COST=1,2,4,8; done
