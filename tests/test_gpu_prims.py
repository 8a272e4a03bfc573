"""The hand-written device primitives of the ingest / layout / build paths
(csrc/prims.cuh: LSD radix sort, exclusive scan, stable select, unique)
against numpy, through dynpr_debug_prims, at the sizes where their code
paths change: empty, single element, tile edges (1024-key small-sort tiles,
2048-item scan / select tiles, 4096-key large-sort tiles, the 8192-tile
rounds of the tile-total scan), the 64-tile
limit of the in-scatter base scan, the 2^18 small / large sort switch, and
multi-pass keys (all digits), constant keys and already-sorted input
(stability is checked through the values)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SIZES = [0, 1, 2, 31, 1023, 1024, 1025, 2047, 2048, 2049, 4095, 4096, 4097, 65535, 65536, 65537,
         (1 << 18), (1 << 18) + 1, 300001, 1 << 21]
# the tile-total scan takes 8192 tiles (of 2048 items) per block round
BIG = [8192 * 2048, 8192 * 2048 + 1, 2 * 8192 * 2048 + 2049]


def _call(dp, op, a, b=None, bits=0, out_dtype=None, out2_dtype=None, n_out=None):
    from paper_2404_08299_b200 import _native as N
    ctx = dp.default_context()
    n = len(a)
    out = np.zeros(max(n_out if n_out is not None else n, 1), out_dtype or a.dtype)
    out2 = np.zeros(max(n, 1), out2_dtype) if out2_dtype is not None else None
    cnt = C.c_uint64()
    rc = N.lib().dynpr_debug_prims(C.c_void_p(ctx.h), op, a.ctypes.data, b.ctypes.data if b is not None else None,
                                   n, bits, out.ctypes.data, out2.ctypes.data if out2 is not None else None,
                                   C.byref(cnt))
    assert rc == 0, N.lib().dynpr_last_error()
    return out, out2, cnt.value


@pytest.mark.parametrize("n", SIZES)
def test_radix_sort_u64_keys(dp, n):
    rng = np.random.default_rng(n)
    for bits, keys in ((49, rng.integers(0, 1 << 49, n, dtype=np.uint64)),
                       (16, rng.integers(0, 1 << 16, n, dtype=np.uint64)),  # many duplicates
                       (40, np.full(n, 12345, np.uint64)),
                       (40, np.arange(n, dtype=np.uint64))):
        out, _, _ = _call(dp, 0, keys, bits=bits)
        assert np.array_equal(out[:n], np.sort(keys))


@pytest.mark.parametrize("n", SIZES)
def test_radix_sort_pairs_is_stable(dp, n):
    rng = np.random.default_rng(n + 7)
    keys = rng.integers(0, 1 << 12, n, dtype=np.uint32)  # duplicates: order of values must be stable
    vals = np.arange(n, dtype=np.uint32)
    ko, vo, _ = _call(dp, 1, keys, vals, bits=12, out2_dtype=np.uint32)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(ko[:n], keys[order])
    assert np.array_equal(vo[:n], vals[order])
    wide = rng.integers(0, 1 << 31, n, dtype=np.uint32)
    ko, vo, _ = _call(dp, 1, wide, vals, bits=31, out2_dtype=np.uint32)
    order = np.argsort(wide, kind="stable")
    assert np.array_equal(ko[:n], wide[order]) and np.array_equal(vo[:n], vals[order])


@pytest.mark.parametrize("n", SIZES + BIG)
def test_exclusive_scan_u64(dp, n):
    rng = np.random.default_rng(n + 11)
    a = rng.integers(0, 1 << 40, n, dtype=np.uint64)
    out, _, total = _call(dp, 2, a)
    ref = np.cumsum(a, dtype=np.uint64) - a if n else a
    assert np.array_equal(out[:n], ref)
    assert total == int(a.sum(dtype=np.uint64)) if n else total == 0


@pytest.mark.parametrize("n", SIZES + BIG)
def test_select_nonzero_indices(dp, n):
    rng = np.random.default_rng(n + 13)
    for density in (0.0, 0.01, 0.5, 1.0):
        f = (rng.random(n) < density).astype(np.uint8)
        out, _, cnt = _call(dp, 3, f, out_dtype=np.uint32)
        ref = np.nonzero(f)[0].astype(np.uint32)
        assert cnt == len(ref) and np.array_equal(out[:cnt], ref)


@pytest.mark.parametrize("n", SIZES)
def test_unique_sorted_u64(dp, n):
    rng = np.random.default_rng(n + 17)
    keys = np.sort(rng.integers(0, max(2, n // 3), n, dtype=np.uint64))
    out, _, cnt = _call(dp, 4, keys)
    ref = np.unique(keys)
    assert cnt == len(ref) and np.array_equal(out[:cnt], ref)
