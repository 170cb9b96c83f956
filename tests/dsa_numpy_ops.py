"""Test double for the distributed suffix array's device steps (paper_1707_03750_b200/dist_sa.py
CudaOps, i.e. the itt_dsa_* kernels of dist.cu), restated with numpy on CPU tensors so the
host driver and its exchanges (gloo, world size 2) run in the CPU suite.  Test infrastructure
only: the product path is CudaOps."""
from __future__ import annotations

import numpy as np
import torch

SAME = 0x80000000
NONE = 0x7FFFFFFF


def _u64(t):
    return t.numpy().view(np.uint64)


def _u32(t):
    return t.numpy().view(np.uint32)


def _t64(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint64).view(np.int64))


def _t32(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint32).view(np.int32))


class NumpyOps:
    device = torch.device("cpu")

    def empty(self, n, dtype):
        return torch.zeros(max(int(n), 0), dtype=dtype)

    def to_device(self, arr, dtype):
        return torch.from_numpy(np.ascontiguousarray(arr)).to(dtype)

    def keys(self, text, np_, lo, cnt, sym_bits, k, rank, rank2, b):
        i = np.arange(lo, lo + cnt, dtype=np.uint64)
        if rank is None:
            t = text.numpy().astype(np.uint64)
            key = np.zeros(cnt, np.uint64)
            for q in range(k):
                idx = i + np.uint64(q)
                c = np.where(idx < np_, t[np.minimum(idx, np_ - 1).astype(np.int64)], 0).astype(np.uint64)
                key = (key << np.uint64(sym_bits)) | c
        else:
            r2 = np.zeros(cnt, np.uint64)
            n2 = 0 if rank2 is None else rank2.numel()
            r2[:n2] = _u32(rank2).astype(np.uint64) + 1
            key = (_u32(rank).astype(np.uint64) << np.uint64(b)) | r2
        return _t64(key), _t32(i.astype(np.uint32))

    def partition(self, a, b, mode, spl_a, spl_b, bounds, P):
        ka = _u64(a)
        if mode == 0:
            kb = _u32(b)
            sa_ = _u64(spl_a) if spl_a is not None else np.zeros(0, np.uint64)
            sb_ = _u32(spl_b) if spl_b is not None else np.zeros(0, np.uint32)
            dest = np.zeros(ka.size, np.int64)
            for x, y in zip(sa_, sb_):
                dest += (x < ka) | ((x == ka) & (y <= kb))
        else:
            pos = (ka & np.uint64(0xFFFFFFFF)).astype(np.int64)
            bd = bounds.numpy()
            dest = np.searchsorted(bd, pos, side="right") - 1
        order = np.argsort(dest, kind="stable")
        counts = np.bincount(dest, minlength=P)[:P].tolist()
        oa = _t64(ka[order])
        ob = _t32(_u32(b)[order]) if b is not None else None
        return oa, ob, [int(c) for c in counts]

    def sort(self, a, b, bits):
        ka = _u64(a)
        mask = np.uint64((1 << bits) - 1) if bits < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
        order = np.argsort(ka & mask, kind="stable")
        a.copy_(_t64(ka[order]))
        b.copy_(_t32(_u32(b)[order]))

    def ids(self, a, b, has_prev, prev, offset):
        ka = _u64(a)
        if ka.size == 0:
            return self.empty(0, torch.int64), 0
        prevs = np.concatenate([[np.uint64(prev)], ka[:-1]])
        flags = ka != prevs
        if not has_prev:
            flags[0] = True
        ids = offset + np.cumsum(flags) - 1
        out = (ids.astype(np.uint64) << np.uint64(32)) | _u32(b).astype(np.uint64)
        return _t64(out), int(flags.sum())

    def scatter(self, p, lo, dst):
        v = _u64(p)
        d = dst.numpy().view(np.uint32)
        d[(v & np.uint64(0xFFFFFFFF)).astype(np.int64) - lo] = (v >> np.uint64(32)).astype(np.uint32)

    def lcp_requests(self, packed, kbase, has_prev, prev):
        v = _u64(packed)
        n = v.size
        prevs = np.concatenate([[np.uint64(prev)], v[:-1]])
        k = np.arange(kbase, kbase + n, dtype=np.uint64)
        a = (k << np.uint64(32)) | (v & np.uint64(0xFFFFFFFF))
        same = (prevs >> np.uint64(32)) == (v >> np.uint64(32))
        bb = (prevs & np.uint64(0xFFFFFFFF)).astype(np.uint32) | np.where(same, SAME, 0).astype(np.uint32)
        if n and not has_prev:
            bb[0] = NONE
        return _t64(a), _t32(bb)

    def kasai(self, text, np_, lo, cnt, req_a, req_b, cap, chunk=64):
        t = text.numpy()
        ra, rb = _u64(req_a), _u32(req_b)
        pos = (ra & np.uint64(0xFFFFFFFF)).astype(np.int64) - lo
        phi = np.zeros(cnt, np.uint32)
        kpos = np.zeros(cnt, np.uint64)
        phi[pos] = rb
        kpos[pos] = ra >> np.uint64(32)
        out = np.zeros(cnt, np.uint64)
        for c0 in range(0, cnt, chunk):
            l, capped = 0, False
            for j in range(c0, min(c0 + chunk, cnt)):
                i = lo + j
                pw = int(phi[j])
                if pw == NONE:
                    v, l, capped = 0, 0, False
                elif pw & SAME:
                    v, l, capped = cap, cap - 1, True
                else:
                    if capped:
                        l = 0
                    while l < cap and i + l < np_ and pw + l < np_ and t[i + l] == t[pw + l]:
                        l += 1
                    v = l
                    capped = False
                    if l > 0:
                        l -= 1
                out[j] = (np.uint64(v) << np.uint64(32)) | kpos[j]
        return _t64(out)

    def sample(self, a, b, s):
        n = a.numel()
        s = min(s, n)
        t = np.arange(s, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        with np.errstate(over="ignore"):
            z = (t ^ (t >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z ^= z >> np.uint64(31)
        j = (z % np.uint64(max(n, 1))).astype(np.int64)
        return _t64(_u64(a)[j]), _t32(_u32(b)[j])

    def copy(self, dst_ptr, src_ptr, nbytes):
        import ctypes
        ctypes.memmove(dst_ptr, src_ptr, nbytes)
