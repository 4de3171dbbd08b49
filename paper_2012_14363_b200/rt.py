"""Node-local multi-process runtime (one process per GPU): bootstrap,
barriers, IPC pointer exchange, datatype Send/Recv with the three transfer
methods of the paper (device / one-shot / staged) selected by the model,
and the distributed halo-exchange plan. Backs the MPI surface (libtempi)."""
from __future__ import annotations

import ctypes as C
import os

from . import _buffer, _check, _capi
from ._capi import lib

DEVICE, ONESHOT, STAGED, DIRECT = 1, 0, 2, 3
AUTO = -1


def init(rank: int, size: int, job: str, device: int = -1, window_bytes: int = 256 << 20,
         host_bytes: int = 256 << 20):
    _check(lib.sp_rt_init(rank, size, job.encode(), device, window_bytes if device >= 0 else 0,
                          host_bytes if device >= 0 else 0))


def finalize():
    _check(lib.sp_rt_finalize())


def rank() -> int:
    v = C.c_int()
    _check(lib.sp_rt_rank(C.byref(v)))
    return v.value


def size() -> int:
    v = C.c_int()
    _check(lib.sp_rt_size(C.byref(v)))
    return v.value


def barrier():
    _check(lib.sp_rt_barrier())


def host_send(dst: int, tag: int, payload: bytes):
    buf = C.create_string_buffer(payload, len(payload))
    _check(lib.sp_rt_host_send(dst, tag, buf, len(payload)))


def host_recv(src: int, tag: int) -> bytes:
    buf = C.create_string_buffer(16)
    n = C.c_int64()
    _check(lib.sp_rt_host_recv(src, tag, buf, 16, C.byref(n)))
    return buf.raw[:n.value]


def exchange_ptr(tensor_or_ptr):
    n = size()
    peers = (C.c_void_p * n)()
    ptr = tensor_or_ptr if isinstance(tensor_or_ptr, int) else tensor_or_ptr.data_ptr()
    _check(lib.sp_rt_exchange_ptr(ptr, peers))
    return [p or 0 for p in peers]


def stream() -> int:
    """cudaStream_t of the runtime (sends, batches, halo plans)"""
    v = C.c_void_p()
    _check(lib.sp_rt_stream(C.byref(v)))
    return v.value or 0


def set_profile(profile):
    _check(lib.sp_rt_set_profile(profile.handle if profile is not None else None))


def choose(ct, count: int) -> int:
    m = C.c_int()
    _check(lib.sp_rt_choose(ct.handle, count, C.byref(m)))
    return m.value


def send(buf, count: int, ct, dest: int, tag: int = 0, method: int = AUTO) -> int:
    a, n, _ = _buffer(buf, False)
    used = C.c_int()
    _check(lib.sp_rt_send(a, n, count, ct.handle, dest, tag, method, C.byref(used)))
    return used.value


def recv(buf, count: int, ct, source: int = -1, tag: int = -1):
    a, n, _ = _buffer(buf, True)
    st = (C.c_int64 * 4)()
    _check(lib.sp_rt_recv(a, n, count, ct.handle, source, tag, st))
    return {"source": st[0], "tag": st[1], "bytes": st[2], "method": st[3]}


def _status(st):
    return {"source": st[0], "tag": st[1], "bytes": st[2], "method": st[3]}


class Request:
    """MPI_Request of sp_rt_isend / sp_rt_irecv; keeps its buffer alive."""

    def __init__(self, handle: int, keep):
        self.handle = handle
        self._keep = keep
        self.status = None

    def test(self) -> bool:
        if self.status is not None:
            return True
        done = C.c_int()
        st = (C.c_int64 * 4)()
        _check(lib.sp_rt_test(self.handle, C.byref(done), st))
        if done.value:
            self.status = _status(st)
        return bool(done.value)

    def wait(self):
        if self.status is None:
            st = (C.c_int64 * 4)()
            _check(lib.sp_rt_wait(self.handle, st))
            self.status = _status(st)
        return self.status


def isend(buf, count: int, ct, dest: int, tag: int = 0, method: int = AUTO) -> Request:
    a, n, _ = _buffer(buf, False)
    h = C.c_uint64()
    _check(lib.sp_rt_isend(a, n, count, ct.handle, dest, tag, method, C.byref(h)))
    return Request(h.value, (buf, ct))


def irecv(buf, count: int, ct, source: int = -1, tag: int = -1) -> Request:
    a, n, _ = _buffer(buf, True)
    h = C.c_uint64()
    _check(lib.sp_rt_irecv(a, n, count, ct.handle, source, tag, C.byref(h)))
    return Request(h.value, (buf, ct))


def waitall(reqs):
    return [r.wait() for r in reqs]


class NeighborW:
    """MPI_Neighbor_alltoallw argument set (built once, called many times):
    sends = [(dest, count, type, byte displacement)], recvs = [(source,
    count, type, byte displacement)]. A call is collective: one typed-copy
    launch per rank, no host barrier."""

    def __init__(self, sends, recvs):
        no, ni = len(sends), len(recvs)
        self._keep = [t for _, _, t, _ in sends] + [t for _, _, t, _ in recvs]
        self.no, self.ni = no, ni
        self.sc = (C.c_int64 * max(no, 1))(*[c for _, c, _, _ in sends])
        self.sd = (C.c_int64 * max(no, 1))(*[d for _, _, _, d in sends])
        self.st = (_capi.sp_type * max(no, 1))(*[t.handle for _, _, t, _ in sends])
        self.dst = (C.c_int * max(no, 1))(*[r for r, _, _, _ in sends])
        self.rc = (C.c_int64 * max(ni, 1))(*[c for _, c, _, _ in recvs])
        self.rd = (C.c_int64 * max(ni, 1))(*[d for _, _, _, d in recvs])
        self.rt = (_capi.sp_type * max(ni, 1))(*[t.handle for _, _, t, _ in recvs])
        self.src = (C.c_int * max(ni, 1))(*[r for r, _, _, _ in recvs])

    def __call__(self, sendbuf, recvbuf):
        sa = sendbuf if isinstance(sendbuf, int) else sendbuf.data_ptr()
        ra = recvbuf if isinstance(recvbuf, int) else recvbuf.data_ptr()
        _check(lib.sp_rt_neighbor_alltoallw(sa, self.sc, self.sd, self.st, self.no, self.dst, ra, self.rc, self.rd,
                                            self.rt, self.ni, self.src))


class NeighborPlan:
    """MPI_Neighbor_alltoallw_init (MPI-4, collective): the exchange of a
    NeighborW argument set compiled once for fixed buffers. start() enqueues
    one signalled launch on the runtime stream (capturable into a CUDA
    graph); wait() completes it."""

    def __init__(self, sends, recvs, sendbuf, recvbuf):
        w = NeighborW(sends, recvs)
        self._w = w
        sa = sendbuf if isinstance(sendbuf, int) else sendbuf.data_ptr()
        ra = recvbuf if isinstance(recvbuf, int) else recvbuf.data_ptr()
        h = C.c_void_p()
        _check(lib.sp_rt_neighbor_alltoallw_init(sa, w.sc, w.sd, w.st, w.no, w.dst, ra, w.rc, w.rd, w.rt, w.ni, w.src,
                                                 C.byref(h)))
        self.handle = h.value

    def start(self):
        _check(lib.sp_nbr_plan_start(self.handle))

    def test(self) -> bool:
        d = C.c_int()
        _check(lib.sp_nbr_plan_test(self.handle, C.byref(d)))
        return bool(d.value)

    def wait(self):
        _check(lib.sp_nbr_plan_wait(self.handle))

    def free(self):
        if self.handle:
            lib.sp_nbr_plan_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def neighbor_alltoallv(sendbuf, sendtype, sends, recvbuf, recvtype, recvs):
    """MPI_Neighbor_alltoallv (collective): sends = [(dest, count,
    displacement in sendtype extents)], recvs = [(source, count,
    displacement in recvtype extents)]"""
    sa = sendbuf if isinstance(sendbuf, int) else sendbuf.data_ptr()
    ra = recvbuf if isinstance(recvbuf, int) else recvbuf.data_ptr()
    no, ni = len(sends), len(recvs)
    I64o, I64i = C.c_int64 * max(no, 1), C.c_int64 * max(ni, 1)
    Io, Ii = C.c_int * max(no, 1), C.c_int * max(ni, 1)
    _check(lib.sp_rt_neighbor_alltoallv(
        sa, I64o(*[c for _, c, _ in sends]), I64o(*[d for _, _, d in sends]), no, Io(*[r for r, _, _ in sends]),
        sendtype.handle, ra, I64i(*[c for _, c, _ in recvs]), I64i(*[d for _, _, d in recvs]), ni,
        Ii(*[r for r, _, _ in recvs]), recvtype.handle))


def neighbor_alltoallw(sendbuf, sends, recvbuf, recvs):
    """one-shot form of NeighborW"""
    NeighborW(sends, recvs)(sendbuf, recvbuf)


def set_chunk(nbytes: int):
    _check(lib.sp_rt_set_chunk(nbytes))


class HaloPlan:
    def __init__(self, cfg, alloc, method: int = 0):
        a, n, _ = _buffer(alloc, True)
        h = C.c_void_p()
        _check(lib.sp_halo_plan_create(C.byref(cfg.c()), a, method, C.byref(h)))
        self.handle = h.value

    def exchange(self, timed: bool = True):
        """one iteration; timed=False only enqueues (DIRECT / FUSED_ASYNC)
        on the runtime stream, so iterations pipeline on the GPU"""
        if not timed:
            _check(lib.sp_halo_plan_exchange(self.handle, None))
            return None
        t = (C.c_double * 4)()
        _check(lib.sp_halo_plan_exchange(self.handle, t))
        return {"pack": t[0], "exchange": t[1], "unpack": t[2], "iteration": t[3]}

    def free(self):
        if self.handle:
            lib.sp_halo_plan_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
