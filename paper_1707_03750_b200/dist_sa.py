"""Distributed suffix array + capped LCP of one trace over G ranks.

The reference builds one suffix tree on one core (suffix_tree.hpp:21-190, via mine.hpp:38-40).
Limits: one B200 takes fewer than 2^32 - 1 suffixes (32-bit SA entries; the radix look-back
words are 64-bit from 2^30 keys on), and its 180 GB hold about 1.5B events with streamed names;
this distributed path takes fewer than 2^31 - 1 suffixes (positions share a u32 with the
same-group flag of the LCP requests).  The suffixes are block-partitioned by text position
across ranks and every doubling round is a global sort of (rank_i, rank_{i+h}) keys:

  1. halo:    rank_{i+h} for own i comes from the owners of [lo+h, hi+h) — one contiguous slice
              per source rank, one all-to-all;
  2. keys:    a = rank_i << b | (rank_{i+h} + 1), b = i          (itt_dsa_keys)
  3. splitters: pseudo-random samples of (a, i), all-gathered, G-1 quantiles
  4. partition by splitter, all-to-all, stable local sort by a    (itt_dsa_partition/_sort);
              sources arrive in rank (= position) order, so ties stay in position order and the
              concatenation of the ranks' slices is the global order by (a, i)
  5. ids:     flags against the previous rank's last key, group counts all-gathered, dense ids
              (itt_dsa_ids); stop when every group is a singleton or h >= cap
  6. route (id, i) back to the owner of i, scatter into the rank array (itt_dsa_partition/_scatter)

LCP (capped at `cap`, as sa.cu): (SA_k, SA_{k-1}, same final group) goes to the owner of SA_k,
Kasai runs over own text positions with the text replicated (itt_dsa_kasai), and (plcp, k)
returns to the owner of sorted position k.  The result on each rank is its slice of SA and LCP
(global sorted positions [kbase, kbase + len)), identical to itt_suffix_array's.

Every per-element step is a hand-written kernel behind the C-ABI (dist.cu); this module is the
host driver: partition bounds, splitter choice, split sizes and convergence.  The exchanges go
through an ``Exchange``: ``TorchExchange`` (torch.distributed — NCCL between B200s, gloo in the
CPU tests) or ``ThreadExchange`` (virtual ranks as threads of one process on one device, for
single-GPU parity tests: the kernels of one virtual rank never wait on another's).
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np
import torch

NONE_PREV = 0x7FFFFFFF
SAMPLES_PER_RANK = 256


def bits_for(v: int) -> int:
    b = 1
    while b < 64 and (v >> b) != 0:
        b += 1
    return b


# --------------------------------------------------------------------------- exchanges
class Exchange:
    rank: int
    size: int

    def all_to_all(self, send: torch.Tensor, counts: list[int]) -> torch.Tensor:
        raise NotImplementedError

    def all_gather_ints(self, vals: list[int]) -> list[list[int]]:
        raise NotImplementedError

    def all_gather_tensor(self, t: torch.Tensor) -> list[torch.Tensor]:
        raise NotImplementedError

    def broadcast(self, t: torch.Tensor, root: int = 0) -> torch.Tensor:
        """t on root (same shape/dtype expected elsewhere: pass a buffer); returns root's data."""
        raise NotImplementedError


class TorchExchange(Exchange):
    """torch.distributed collectives (NCCL for CUDA tensors, gloo for CPU tensors)."""

    def __init__(self, group=None, device: torch.device | None = None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.device = device or torch.device("cpu")

    def _counts(self, counts: list[int]) -> list[int]:
        c = torch.tensor(counts, dtype=torch.int64, device=self.device)
        r = torch.empty_like(c)
        self.dist.all_to_all_single(r, c, group=self.group)
        return r.cpu().tolist()

    def all_to_all(self, send, counts):
        rc = self._counts(counts)
        out = torch.empty(sum(rc), dtype=send.dtype, device=send.device)
        self.dist.all_to_all_single(out, send.contiguous(), output_split_sizes=rc, input_split_sizes=list(counts),
                                    group=self.group)
        self._settle(out)
        return out

    @staticmethod
    def _settle(t):
        # NCCL orders the collective only against torch's current stream; the device steps run on
        # the library context's own stream, so the host waits for the result here
        if t.is_cuda:
            torch.cuda.current_stream(t.device).synchronize()

    def all_gather_ints(self, vals):
        t = torch.tensor(vals, dtype=torch.int64, device=self.device)
        out = [torch.empty_like(t) for _ in range(self.size)]
        self.dist.all_gather(out, t, group=self.group)
        return [o.cpu().tolist() for o in out]

    def all_gather_tensor(self, t):
        n = self.all_gather_ints([t.numel()])
        m = max(x[0] for x in n)
        pad = torch.zeros(m, dtype=t.dtype, device=t.device)
        pad[: t.numel()] = t
        out = [torch.empty_like(pad) for _ in range(self.size)]
        self.dist.all_gather(out, pad, group=self.group)
        return [o[: x[0]] for o, x in zip(out, n)]

    def broadcast(self, t, root=0):
        self.dist.broadcast(t, src=root, group=self.group)
        self._settle(t)
        return t


class _Board:
    def __init__(self, size):
        self.size = size
        self.slots = [None] * size
        self.barrier = threading.Barrier(size)


class ThreadExchange(Exchange):
    """Virtual ranks as threads of one process (one device): a shared board + barriers."""

    def __init__(self, board: _Board, rank: int):
        self.board = board
        self.rank = rank
        self.size = board.size

    @staticmethod
    def group(size: int) -> list["ThreadExchange"]:
        b = _Board(size)
        return [ThreadExchange(b, r) for r in range(size)]

    def _post(self, obj):
        b = self.board
        b.slots[self.rank] = obj
        b.barrier.wait()
        got = list(b.slots)
        b.barrier.wait()  # everyone has read the board; the posted buffers may be released
        return got

    def all_to_all(self, send, counts):
        offs = np.concatenate([[0], np.cumsum(counts)]).tolist()
        if send.is_cuda:
            torch.cuda.synchronize(send.device)
        b = self.board
        b.slots[self.rank] = (send, offs)
        b.barrier.wait()
        pieces = [b.slots[q][0][b.slots[q][1][self.rank]: b.slots[q][1][self.rank + 1]] for q in range(self.size)]
        out = torch.cat(pieces) if pieces else send[:0]
        if out.is_cuda:
            torch.cuda.synchronize(out.device)
        b.barrier.wait()
        return out

    def all_gather_ints(self, vals):
        return [list(v) for v in self._post(list(vals))]

    def all_gather_tensor(self, t):
        got = self._post(t)
        return [g.clone() for g in got]

    def broadcast(self, t, root=0):
        if t.is_cuda:
            torch.cuda.synchronize(t.device)
        got = self._post(t if self.rank == root else None)
        if self.rank != root:
            t.copy_(got[root])
            if t.is_cuda:
                torch.cuda.synchronize(t.device)
        self.board.barrier.wait()
        return t


# --------------------------------------------------------------------------- device steps
class CudaOps:
    """The per-rank device steps: hand-written kernels behind itt_dsa_* (dist.cu).  Tensors are
    int64 / int32 torch tensors on the context's device (reinterpreted as u64 / u32)."""

    def __init__(self, ctx):
        from . import cuda
        self.ctx = ctx
        self.L = cuda.lib()
        self.device = torch.device("cuda", ctx.device)

    def empty(self, n, dtype):
        return torch.empty(max(int(n), 0), dtype=dtype, device=self.device)

    @staticmethod
    def _p(t):
        return C.c_void_p(t.data_ptr()) if t is not None and t.numel() else None

    def keys(self, text, np_, lo, cnt, sym_bits, k, rank, rank2, b):
        a = self.empty(cnt, torch.int64)
        v = self.empty(cnt, torch.int32)
        n2 = 0 if rank2 is None else rank2.numel()
        self.ctx._check(self.L.itt_dsa_keys(self.ctx.h, self._p(text), np_, lo, cnt, sym_bits, k, self._p(rank),
                                            self._p(rank2), n2, b, self._p(a), self._p(v)))
        return a, v

    def partition(self, a, b, mode, spl_a, spl_b, bounds, P):
        cnt = a.numel()
        oa = self.empty(cnt, torch.int64)
        ob = self.empty(cnt, torch.int32) if b is not None else None
        counts = (C.c_uint64 * P)()
        nspl = 0 if spl_a is None else spl_a.numel()
        self.ctx._check(self.L.itt_dsa_partition(self.ctx.h, self._p(a), self._p(b), cnt, mode, self._p(spl_a),
                                                 self._p(spl_b), nspl, self._p(bounds), P, self._p(oa), self._p(ob),
                                                 counts))
        return oa, ob, [int(x) for x in counts]

    def sort(self, a, b, bits):
        self.ctx._check(self.L.itt_dsa_sort(self.ctx.h, self._p(a), self._p(b), a.numel(), bits))

    def ids(self, a, b, has_prev, prev, offset, want_out=True):
        out = self.empty(a.numel(), torch.int64)
        ng = C.c_uint64()
        self.ctx._check(self.L.itt_dsa_ids(self.ctx.h, self._p(a), self._p(b), a.numel(), int(has_prev), prev, offset,
                                           self._p(out), C.byref(ng)))
        return out, int(ng.value)

    def scatter(self, p, lo, dst):
        self.ctx._check(self.L.itt_dsa_scatter(self.ctx.h, self._p(p), p.numel(), lo, self._p(dst)))

    def lcp_requests(self, packed, kbase, has_prev, prev):
        a = self.empty(packed.numel(), torch.int64)
        b = self.empty(packed.numel(), torch.int32)
        self.ctx._check(self.L.itt_dsa_lcp_requests(self.ctx.h, self._p(packed), packed.numel(), kbase, int(has_prev),
                                                    prev, self._p(a), self._p(b)))
        return a, b

    def kasai(self, text, np_, lo, cnt, req_a, req_b, cap):
        out = self.empty(cnt, torch.int64)
        self.ctx._check(self.L.itt_dsa_kasai(self.ctx.h, self._p(text), np_, lo, cnt, self._p(req_a), self._p(req_b),
                                             cap, self._p(out)))
        return out

    def sample(self, a, b, s):
        s = min(s, a.numel())
        oa = self.empty(s, torch.int64)
        ob = self.empty(s, torch.int32)
        self.ctx._check(self.L.itt_dsa_sample(self.ctx.h, self._p(a), self._p(b), a.numel(), s, self._p(oa),
                                              self._p(ob)))
        return oa, ob

    def to_device(self, arr: np.ndarray, dtype):
        return torch.from_numpy(np.ascontiguousarray(arr)).to(dtype=dtype, device=self.device)

    def copy(self, dst_ptr, src_ptr, nbytes):
        if torch.cuda.is_available():
            torch.cuda.synchronize(self.device)  # torch-side producers of src / consumers of dst
        self.ctx._check(self.L.itt_memcpy(self.ctx.h, C.c_void_p(dst_ptr), C.c_void_p(src_ptr), nbytes))


# --------------------------------------------------------------------------- driver
@dataclass
class DistSA:
    """This rank's slice of the global suffix array: sorted positions [kbase, kbase + len(sa))."""
    kbase: int
    sa: torch.Tensor            # int32 (u32 positions)
    lcp: torch.Tensor | None    # int32, min(lcp, cap) — exact when the doubling fully converged
    rounds: int
    groups: int
    h_final: int
    cap: int


def _u64(x: int) -> int:
    return x & 0xFFFFFFFFFFFFFFFF


def _prev_nonempty(table: list[list[int]], r: int):
    """(has_prev, value) of the last element of the nearest non-empty rank before r.
    table[q] = [count, last_value]."""
    for q in range(r - 1, -1, -1):
        if table[q][0] > 0:
            return True, _u64(table[q][1])
    return False, 0


def _splitters(ex: Exchange, ops, a, v, P):
    sa_, sb_ = ops.sample(a, v, SAMPLES_PER_RANK)
    ga = ex.all_gather_tensor(sa_)
    gb = ex.all_gather_tensor(sb_)
    ka = np.concatenate([g.cpu().numpy().view(np.uint64) for g in ga])
    kb = np.concatenate([g.cpu().numpy().view(np.uint32) for g in gb])
    if ka.size == 0:
        ka = np.zeros(1, np.uint64)
        kb = np.zeros(1, np.uint32)
    order = np.lexsort((kb, ka))
    ka, kb = ka[order], kb[order]
    pick = [min(ka.size - 1, (q * ka.size) // P) for q in range(1, P)]
    return (ops.to_device(ka[pick].view(np.int64), torch.int64), ops.to_device(kb[pick].view(np.int32), torch.int32))


def _sample_sort(ex: Exchange, ops, a, v, key_bits):
    """Global sort by (a, position): returns this rank's slice of the sorted sequence."""
    P = ex.size
    if P == 1:
        ops.sort(a, v, key_bits)
        return a, v
    spl_a, spl_b = _splitters(ex, ops, a, v, P)
    oa, ob, counts = ops.partition(a, v, 0, spl_a, spl_b, None, P)
    del a, v
    ra = ex.all_to_all(oa, counts)
    rb = ex.all_to_all(ob, counts)
    del oa, ob
    ops.sort(ra, rb, key_bits)
    return ra, rb


def suffix_array_dist(ex: Exchange, ops, text: torch.Tensor, n: int, term: int, cap: int = 0xFFFFFFFF,
                      want_lcp: bool = True) -> DistSA:
    """SPMD: every rank calls this with the replicated text (tokens + [term], int32, tokens in
    [0, term)).  cap = max L_max + 1 for mining (sa.cu's capped doubling); 0xFFFFFFFF = full."""
    P, r = ex.size, ex.rank
    np_ = n + 1
    if np_ >= 0x7FFFFFFF:
        raise ValueError("distributed suffix array: n + 1 must stay below 2^31 - 1")
    bounds_l = [q * np_ // P for q in range(P + 1)]
    lo, hi = bounds_l[r], bounds_l[r + 1]
    cnt = hi - lo
    bounds = ops.to_device(np.array(bounds_l, np.int64), torch.int64)
    sym_bits = bits_for(term)
    k = max(1, 64 // sym_bits)
    a, v = ops.keys(text, np_, lo, cnt, sym_bits, k, None, None, 0)
    key_bits = min(64, sym_bits * k)
    h = k
    rounds = 0
    while True:
        a, v = _sample_sort(ex, ops, a, v, key_bits)
        last = int(a[-1].item()) if a.numel() else 0
        table = ex.all_gather_ints([a.numel(), last])
        has_prev, prev = _prev_nonempty(table, r)
        _, ng = ops.ids(a, v, has_prev, prev, 0)
        counts = ex.all_gather_ints([ng])
        G = sum(c[0] for c in counts)
        offset = sum(counts[q][0] for q in range(r))
        packed, _ = ops.ids(a, v, has_prev, prev, offset)
        del a, v
        if G == np_ or h >= cap:
            break
        # (id, i) back to the owner of i
        oa, _, cts = ops.partition(packed, None, 1, None, None, bounds, P)
        del packed
        back = ex.all_to_all(oa, cts)
        del oa
        rank = ops.empty(cnt, torch.int32)
        ops.scatter(back, lo, rank)
        del back
        # halo: ranks of positions [lo + h, min(hi + h, np_)) from their owners (one slice per source)
        sends = []
        for q in range(P):
            s0 = max(bounds_l[q] + h, lo)
            e0 = min(bounds_l[q + 1] + h, hi, np_)
            sends.append((s0, max(0, e0 - s0)))
        first = next((s0 for s0, c in sends if c > 0), lo)
        tot = sum(c for _, c in sends)
        rank2 = ex.all_to_all(rank[first - lo: first - lo + tot], [c for _, c in sends])
        b = bits_for(G)
        a, v = ops.keys(text, np_, lo, cnt, sym_bits, k, rank, rank2, b)
        del rank, rank2
        key_bits = bits_for(G - 1) + b
        rounds += 1
        if h * 2 > 0xFFFFFFFF:
            break
        h *= 2
    table = ex.all_gather_ints([packed.numel(), int(packed[-1].item()) if packed.numel() else 0])
    kbase = sum(table[q][0] for q in range(r))
    sa = (packed & 0xFFFFFFFF).to(torch.int32) if packed.numel() else ops.empty(0, torch.int32)
    eff_cap = 0xFFFFFFFF if G == np_ else cap
    lcp = None
    if want_lcp:
        has_prev, prev = _prev_nonempty(table, r)
        ra, rb = ops.lcp_requests(packed, kbase, has_prev, prev)
        oa, ob, cts = ops.partition(ra, rb, 1, None, None, bounds, P)
        del ra, rb
        qa = ex.all_to_all(oa, cts)
        qb = ex.all_to_all(ob, cts)
        del oa, ob
        out = ops.kasai(text, np_, lo, cnt, qa, qb, eff_cap)
        del qa, qb
        kb_l = [sum(table[q][0] for q in range(p)) for p in range(P + 1)]
        kbounds = ops.to_device(np.array(kb_l, np.int64), torch.int64)
        oa, _, cts = ops.partition(out, None, 1, None, None, kbounds, P)
        del out
        back = ex.all_to_all(oa, cts)
        lcp = ops.empty(packed.numel(), torch.int32)
        ops.scatter(back, kbase, lcp)
    return DistSA(kbase=kbase, sa=sa, lcp=lcp, rounds=rounds, groups=G, h_final=h, cap=eff_cap)


def gather_to_root(ex: Exchange, t: torch.Tensor, root: int = 0) -> torch.Tensor | None:
    """Concatenate every rank's slice on `root` (all-to-all with only the root receiving)."""
    counts = [t.numel() if q == root else 0 for q in range(ex.size)]
    out = ex.all_to_all(t, counts)
    return out if ex.rank == root else None


def run_virtual(P: int, fn):
    """Run fn(exchange, rank) on P virtual ranks (threads); returns the per-rank results."""
    exs = ThreadExchange.group(P)
    res = [None] * P
    err = []

    def body(q):
        try:
            res[q] = fn(exs[q], q)
        except BaseException as e:  # noqa: BLE001 (re-raised below)
            err.append(e)
            exs[q].board.barrier.abort()

    ts = [threading.Thread(target=body, args=(q,)) for q in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if err:
        raise err[0]
    return res


# --------------------------------------------------------------------------- analyze over G ranks
class DistributedSAProvider:
    """itt_analyze's suffix-array hook (itt_analyze_opts.sa_provider) on the root rank: the root
    analyzes the trace (ingest, dictionary, tokens, then mining / matching / aggregates); the
    suffix array and LCP in between are built by all G ranks.  Per analyze the root broadcasts
    (n, term, cap) and the tokens (the text is replicated: 4 B per token), every rank runs
    suffix_array_dist, and the slices are gathered back into the library's sa / lcp buffers.
    The other ranks sit in serve() until the root calls stop()."""

    def __init__(self, ex: Exchange, ops, root: int = 0):
        self.ex, self.ops, self.root = ex, ops, root
        self.last: DistSA | None = None

    def _header(self, vals):
        t = torch.tensor(vals, dtype=torch.int64, device=self.ops.device)
        return self.ex.broadcast(t, self.root).cpu().tolist()

    def _round(self, n, term, cap, text):
        r = suffix_array_dist(self.ex, self.ops, text, n, term, cap)
        self.last = r
        sa = gather_to_root(self.ex, r.sa, self.root)
        lcp = gather_to_root(self.ex, r.lcp, self.root)
        return sa, lcp

    def __call__(self, tok_ptr, n, term, cap, sa_ptr, lcp_ptr):
        self._header([n, term, cap])
        text = self.ops.empty(n + 1, torch.int32)
        self.ops.copy(text.data_ptr(), tok_ptr, (n + 1) * 4)
        self.ex.broadcast(text, self.root)
        sa, lcp = self._round(n, term, cap, text)
        self.ops.copy(sa_ptr, sa.data_ptr(), (n + 1) * 4)
        self.ops.copy(lcp_ptr, lcp.data_ptr(), (n + 1) * 4)

    def serve(self):
        """Non-root ranks: take part in every distributed suffix array until stop()."""
        while True:
            n, term, cap = self._header([0, 0, 0])
            if n < 0:
                return
            text = self.ops.empty(n + 1, torch.int32)
            self.ex.broadcast(text, self.root)
            self._round(n, term, cap, text)

    def stop(self):
        self._header([-1, 0, 0])

