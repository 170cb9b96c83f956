"""The distributed suffix array driven natively (csrc/dist_driver.cu, itt_comm_* / itt_dsa_*).

SURVEY §8(e), C5: one trace's suffix array over G ranks.  The exchanges run in the library on the
context's stream — NCCL between GPUs (grouped ncclSend/ncclRecv all-to-alls, ncclAllGather,
ncclBroadcast) or virtual ranks (threads of one process on one device, for tests) — so Python
only sets the communicators up.  dist_sa.py is the same algorithm in Python (its numpy / gloo
tests run on CPU); this module is the production path:

    comm = Comm.nccl(ctx, world, rank, uid)              # uid from Comm.unique_id() on rank 0, broadcast
    part = build(ctx, comm, text, n, term, cap)          # this rank's slice of SA / LCP
    prov = Provider(ctx_dsa, comm, root=0)               # itt_analyze over G ranks:
    ctx.analyze_raw(recs, loops, native_provider=prov)   #   root
    prov.serve()                                         #   every other rank, until prov.stop() on the root
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

from . import abi
from .cuda import Context, IttError, lib


class Comm:
    def __init__(self, handle: int):
        self.handle = handle

    @staticmethod
    def unique_id() -> bytes:
        uid = (C.c_uint8 * 128)()
        rc = lib().itt_comm_nccl_unique_id(uid)
        if rc:
            raise IttError(rc, "ncclGetUniqueId failed")
        return bytes(uid)

    @staticmethod
    def nccl(ctx: Context, nranks: int, rank: int, uid: bytes) -> "Comm":
        h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        ctx._check(lib().itt_comm_create_nccl(ctx.h, nranks, rank, buf, C.byref(h)))
        return Comm(h.value)

    @staticmethod
    def local(nranks: int) -> list["Comm"]:
        hs = (C.c_void_p * nranks)()
        rc = lib().itt_comm_create_local(nranks, hs)
        if rc:
            raise IttError(rc, "itt_comm_create_local failed")
        return [Comm(hs[i]) for i in range(nranks)]

    def abort(self):
        lib().itt_comm_abort(C.c_void_p(self.handle))

    def close(self):
        if self.handle:
            lib().itt_comm_destroy(C.c_void_p(self.handle))
            self.handle = None


@dataclass
class Slice:
    """This rank's slice: sorted positions [kbase, kbase + count) of the suffix array (device)."""
    kbase: int
    count: int
    sa_ptr: int
    lcp_ptr: int
    info: abi.itt_dsa_info
    ctx: Context

    def free(self):
        for p in (self.sa_ptr, self.lcp_ptr):
            if p:
                lib().itt_device_free(self.ctx.h, C.c_void_p(p))
        self.sa_ptr = self.lcp_ptr = 0


def build(ctx: Context, comm: Comm, text_ptr: int, n: int, term: int, cap: int = 0xFFFFFFFF, want_lcp: bool = True) -> Slice:
    """itt_dsa_build: SPMD over the communicator's ranks; text = tokens + [term] on this rank's device."""
    sa, lcp = C.c_void_p(), C.c_void_p()
    kbase, count = C.c_uint64(), C.c_uint64()
    info = abi.itt_dsa_info()
    ctx._check(lib().itt_dsa_build(ctx.h, C.c_void_p(comm.handle), C.c_void_p(text_ptr), n, term, cap, 1 if want_lcp else 0,
                                   C.byref(sa), C.byref(lcp) if want_lcp else None, C.byref(kbase), C.byref(count),
                                   C.byref(info)))
    return Slice(kbase.value, count.value, sa.value or 0, lcp.value or 0, info, ctx)


class Provider:
    """itt_analyze's sa_provider over G ranks (root: pass as analyze_raw(native_provider=...))."""

    def __init__(self, ctx: Context, comm: Comm, root: int = 0):
        self.ctx, self.comm = ctx, comm
        h = C.c_void_p()
        ctx._check(lib().itt_dsa_provider_create(ctx.h, C.c_void_p(comm.handle), root, C.byref(h)))
        self.handle = h.value

    def serve(self):
        rc = lib().itt_dsa_serve(C.c_void_p(self.handle))
        if rc:
            raise IttError(rc, self.ctx_error())

    def stop(self):
        self.ctx._check(lib().itt_dsa_stop(C.c_void_p(self.handle)))

    def last_info(self) -> abi.itt_dsa_info:
        info = abi.itt_dsa_info()
        lib().itt_dsa_last_info(C.c_void_p(self.handle), C.byref(info))
        return info

    def ctx_error(self) -> str:
        return lib().itt_last_error(self.ctx.h).decode()

    def close(self):
        if self.handle:
            lib().itt_dsa_provider_destroy(C.c_void_p(self.handle))
            self.handle = None


def run_local(P: int, fn):
    """fn(rank, comm) on P virtual ranks (threads; ctypes releases the GIL inside the library)."""
    comms = Comm.local(P)
    res, err = [None] * P, []

    def body(q):
        try:
            res[q] = fn(q, comms[q])
        except BaseException as e:  # noqa: BLE001 (re-raised below)
            err.append(e)
            comms[q].abort()

    ts = [threading.Thread(target=body, args=(q,)) for q in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for cm in comms:
        cm.close()
    if err:
        raise err[0]
    return res
