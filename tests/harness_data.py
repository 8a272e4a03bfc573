"""Deterministic input files for the loader / harness tests (no reference
data is read at run time: /root/reference does not exist on the GPU box)."""
import numpy as np


def write_temporal_stream(path, n_vertices=1500, entries=10000, seed=3, shuffle_ids=True, unsorted=False):
    """A synthetic SNAP-layout temporal stream (`src dst unixts`, `#`
    comments) like the reference's fixture: uniform random pairs with
    non-decreasing timestamps and raw ids drawn from a sparse id space."""
    rng = np.random.default_rng(seed)
    raw = rng.choice(10 * n_vertices, n_vertices, replace=False) if shuffle_ids else np.arange(n_vertices)
    s = raw[rng.integers(0, n_vertices, entries)]
    d = raw[rng.integers(0, n_vertices, entries)]
    ts = 1217567877 + np.cumsum(rng.integers(0, 3, entries))
    if unsorted:
        ts = ts[rng.permutation(entries)]
    with open(path, "w") as f:
        f.write("# synthetic temporal network, SNAP layout\n# src dst unixts\n")
        f.write(f"# {entries} temporal edges\n")
        for a, b, t in zip(s.tolist(), d.tolist(), ts.tolist()):
            f.write(f"{a} {b} {t}\n")
    return path


def write_matrix_market(path, n, pairs, seed=5, symmetry="general", weights=False):
    """A coordinate MatrixMarket file with `pairs` uniform random entries
    (1-based, duplicates allowed)."""
    rng = np.random.default_rng(seed)
    i = rng.integers(1, n + 1, pairs)
    j = rng.integers(1, n + 1, pairs)
    field = "real" if weights else "pattern"
    with open(path, "w") as f:
        f.write(f"%%MatrixMarket matrix coordinate {field} {symmetry}\n% generated\n")
        f.write(f"{n} {n} {pairs}\n")
        for a, b in zip(i.tolist(), j.tolist()):
            f.write(f"{a} {b} 1.5\n" if weights else f"{a} {b}\n")
    return path
