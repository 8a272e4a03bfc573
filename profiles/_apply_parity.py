import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, paper_2404_08299_b200 as dp, oracle
O = oracle.Oracle("ref")
src, dst = O.rmat_edges(18, 16 << 18)
og = O.add_self_loops(O.build_csr((src, dst), 1 << 18))
g = dp.CsrGraph.from_csr(og.n, *og.csr()); gt = dp.transpose(g)
ok = True
for seed in range(6):
    dels, ins = O.generate_random_batch(og, [10, 4000, 40000][seed % 3], 0.8, seed)
    og2, _, _ = O.apply_batch(og, dels, ins)
    g2, gt2 = dp.apply_batch_pair(g, gt, dp.BatchUpdate(dels, ins))
    off, tgt = og2.csr(); offT, tgtT = O.transpose(og2).csr()
    r = (np.array_equal(g2.targets, tgt), np.array_equal(gt2.targets, tgtT), np.array_equal(g2.offsets, off))
    ok &= all(r)
    print(seed, r)
print("ALL OK" if ok else "MISMATCH")
