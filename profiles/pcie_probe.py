"""Pinned host<->device copy rates on the box (the e2e floor in DESIGN §5b):
1.25 GB (RMAT-24 transpose CSR) H2D and 134 MB D2H, best of 5, CUDA events."""
import json
import torch

out = {}
for name, nbytes, h2d in (("h2d_1.25GB", 1_254_000_000, True), ("d2h_134MB", 134_217_728, False)):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        (d.copy_(h, non_blocking=True) if h2d else h.copy_(d, non_blocking=True))
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    out[name] = {"ms": best, "GB_per_s": nbytes / best / 1e6}
print(json.dumps(out))
