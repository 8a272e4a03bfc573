"""Golden report digests for the harness parity tests, generated FROM THE
REFERENCE ITSELF (oracle/_ref: runExperiment + emitReport of the unmodified
library) on the deterministic synthetic inputs of tests/harness_data.py, so
tests/test_gpu_harness.py can check the device harness's report bytes even
where the reference library is not available.

    python tests/golden/make_harness_golden.py    -> harness_golden.json
"""
import ctypes as C
import hashlib
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402
from harness_data import write_matrix_market, write_temporal_stream  # noqa: E402

# name -> (input writer kwargs, spec fields); mirrors test_gpu_harness.py
CASES = {
    "temporal_criterion9": ("temporal", dict(), dict(mode=1, sizes=["1e-3"], approaches=[0, 1, 2, 3, 4], seed=1)),
    "random_general": ("mtx", dict(n=2000, pairs=16000, symmetry="general", seed=13),
                       dict(mode=2, sizes=["1e-3", "1e-2"], approaches=[0, 1, 2, 3, 4], seed=7, repetitions=2)),
}


def spec_struct(path, f):
    from paper_2404_08299_b200 import _native as N
    c = N.ExperimentSpec()
    N.lib().dynpr_experiment_spec_default(C.byref(c))
    sizes = [s.encode() for s in f["sizes"]]
    keep = [(C.c_char_p * max(len(sizes), 1))(*sizes), (C.c_int32 * len(f["approaches"]))(*f["approaches"]),
            path.encode()]
    c.batch_size_specs, c.approaches, c.graph_path = keep
    c.n_batch_size_specs = len(sizes)
    c.n_approaches = len(f["approaches"])
    c.mode = f["mode"]
    c.seed = f["seed"]
    c.repetitions = f.get("repetitions", 1)
    c.record_timing = 0
    return c, keep


def make_input(kind, kw, d):
    if kind == "temporal":
        return write_temporal_stream(os.path.join(d, "temporal-10k.txt"), **kw)
    return write_matrix_market(os.path.join(d, "rb-%s.mtx" % kw["symmetry"]), kw["n"], kw["pairs"], seed=kw["seed"],
                               symmetry=kw["symmetry"])


def main():
    R = oracle.Oracle("ref")
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for name, (kind, kw, f) in CASES.items():
            path = make_input(kind, kw, d)
            c, keep = spec_struct(path, f)
            rep = os.path.join(d, name + ".csv")
            R.run_experiment(c, 0, rep)
            data = open(rep, "rb").read()
            out[name] = {"md5": hashlib.md5(data).hexdigest(), "bytes": len(data)}
    with open(os.path.join(HERE, "harness_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(out)


if __name__ == "__main__":
    main()
