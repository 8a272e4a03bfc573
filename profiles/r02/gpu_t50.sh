# pull-only frontier kernels (timing experiment, results not checked)
set -x
for d in . _ab_pullonly; do echo "== $d"; DYNPR_PKG_ROOT=$PWD/$d timeout 300 python profiles/dfp_iter_probe.py 24 1e-4 2>&1 | grep -A16 '^dfp'; done
