# TMA gather4 vs LDG random-gather microbenchmark
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_tma profiles/microbench_tma_gather.cu -lcuda
timeout 300 /tmp/mb_tma
