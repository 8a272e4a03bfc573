"""Static device ms (min / median of 7 warm solves) of RMAT-S graphs for
several package builds (directories holding paper_2404_08299_b200/ with its
built library), one process per (build, scale), builds interleaved."""
import os, subprocess, sys
CHILD = r'''
import sys, statistics
sys.path.insert(0, sys.argv[1])
import paper_2404_08299_b200 as dp
g = dp.rmat_graph(int(sys.argv[2])); gt = dp.transpose(g); dp.prepare(gt, g)
ms = [dp.static_pagerank(gt, g).device_ms for _ in range(8)][1:]
print("%.3f %.3f" % (min(ms), statistics.median(ms)))
'''
scales = sys.argv[1].split(",")
dirs = sys.argv[2:]
for scale in scales:
    for rep in range(2):
        for spec in dirs:  # DIR or DIR:VAR=value
            d, _, kv = spec.partition(":")
            env = dict(os.environ)
            for item in filter(None, kv.split("+")):  # VAR=value[+VAR2=value2]
                k, v = item.split("=")
                env[k] = v
            out = subprocess.run([sys.executable, "-c", CHILD, os.path.abspath(d), scale], capture_output=True,
                                 text=True, cwd="/tmp", env=env)
            print(scale, spec, out.stdout.strip() or out.stderr[-300:], flush=True)
