nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cif profiles/r02/cond_if_probe.cu && timeout 60 /tmp/cif
