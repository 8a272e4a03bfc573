"""Cold vs warm ingest + layout on a Kronecker graph (configs[3]).  Prints
per-repetition apply_batch_pair / prepare times and free device memory;
run with DYNPR_ALLOC_DEBUG=1 to see slow pool growth; KRON=0 for RMAT.
    python profiles/kron_ingest_probe.py [scale] [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ROOT = os.environ.get("DYNPR_PKG_ROOT", ROOT)  # (A/B: another build of the package)
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_2404_08299_b200 as dp  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3


def free_gb():
    return torch.cuda.mem_get_info()[0] / 2**30


g0 = dp.kronecker_graph(scale) if os.environ.get("KRON", "1") == "1" else dp.rmat_graph(scale)
gt0 = dp.transpose(g0)
print("built n=%d m=%d free=%.1f GB" % (g0.vertex_count, g0.edge_count, free_gb()), flush=True)
t0 = time.perf_counter()
lay0 = dp.prepare(gt0, g0)
print("base prepare %.1f ms (device %.1f) free=%.1f GB" % ((time.perf_counter() - t0) * 1e3, lay0, free_gb()),
      flush=True)
m = g0.edge_count
size = dp.batch_size_from_fraction(1e-4, m)
for r in range(reps):
    b = dp.generate_random_batch(g0, size, 0.8, dp.derive_seed(42, 1000003 + r))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g, gt = dp.apply_batch_pair(g0, gt0, b)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    lay = dp.prepare(gt, g)
    t2 = time.perf_counter()
    print("rep %d: apply_batch_pair %.1f ms, prepare %.1f ms (device %.1f), free=%.1f GB"
          % (r, (t1 - t0) * 1e3, (t2 - t1) * 1e3, lay, free_gb()), flush=True)
    del g, gt
