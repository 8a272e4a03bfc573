set -x
timeout 600 python -m pytest tests/test_gpu_graph.py -q -x -k "kronecker or rmat" 2>&1 | tail -2
timeout 900 python profiles/grid_ab.py 24 -:-,2:3,2:4,1:3,3:2,2:5,1:2,2:2,3:3
timeout 900 python profiles/grid_ab.py 26 -:-,2:3,2:4,3:3,1:3
timeout 900 python profiles/grid_ab.py k25 -:-,2:3,2:4,3:3
DYNPR_SWEEP=split timeout 900 python profiles/grid_ab.py 23 -:-,2:3,2:4
DYNPR_SWEEP=split timeout 900 python profiles/grid_ab.py 22 -:-,2:3,2:4
