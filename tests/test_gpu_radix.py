"""The onesweep radix sort (K4/K5 behind the suffix array and the (start,row) order,
ingest.hpp:396-400): stable LSD sort of (u32 key, u32 value) pairs, checked against numpy's stable
argsort, and past 2^30 pairs where one digit holds more than 2^30 keys (the look-back words then
switch from 32-bit to 64-bit: a 30-bit count field overflowed into the flag bits before)."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,bits,skew", [(1, 8, 0), (4095, 8, 0), (4097, 12, 0), (100_003, 32, 0),
                                         (1_000_000, 20, 1), (3_000_017, 32, 1), (262_144, 9, 2)])
def test_sort_pairs_matches_stable_argsort(ctx, n, bits, skew):
    rng = np.random.default_rng(n + bits)
    if skew == 0:
        keys = rng.integers(0, 1 << bits, n, dtype=np.uint64).astype(np.uint32)
    elif skew == 1:  # mostly one key: long runs of one digit
        keys = np.where(rng.random(n) < 0.97, 7, rng.integers(0, 1 << bits, n)).astype(np.uint32)
    else:  # sorted runs (the SA's group ids)
        keys = np.sort(rng.integers(0, 1 << bits, n)).astype(np.uint32)[::-1].copy()
    vals = np.arange(n, dtype=np.uint32)
    k, v = ctx.radix_sort_pairs(keys, vals, 0, bits)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(k, keys[order])
    assert np.array_equal(v, vals[order])


def test_sort_beyond_2_pow_30_pairs(ctx):
    """2^30 + 2^20 pairs, digit 0 of pass 0 holds ~2^30 keys: the per-digit inclusive count of the
    last tiles exceeds 2^30 (radix.cuh Status<u32> cannot hold it; Status<u64> is used)."""
    import torch
    dev = torch.device("cuda", 0)
    n = (1 << 30) + (1 << 20)
    idx = torch.arange(n, dtype=torch.int64, device=dev)
    keys = torch.zeros(n, dtype=torch.int32, device=dev)
    keys[idx % 4099 == 0] = 3          # a sprinkling of other digits (the pass is not trivial)
    keys[idx % 65537 == 11] = 200
    keys[n - 5:] = 1
    del idx
    vals = torch.arange(n, dtype=torch.int32, device=dev)
    want_k, want_perm = torch.sort(keys, stable=True)
    torch.cuda.synchronize()
    ctx.radix_sort_device(keys.data_ptr(), vals.data_ptr(), n, 0, 8)
    torch.cuda.synchronize()
    assert torch.equal(keys, want_k)
    assert torch.equal(vals, want_perm.to(torch.int32))
