#!/bin/bash
# configs[3] on one B200: Kronecker/RMAT scale-27 (~2.1 B edges) Static + DF-P
# with a bounded reference CPU sample.  Run under gpurun with a timeout.
cd "$(dirname "$0")/.."
timeout 1500 python profiles/configs_bench.py --configs 3 --kron-scale ${1:-27} --out gpurun_out/configs_kron.json
