"""3D halo exchange (paper §6.4; reference halo.hpp) on B200.

    HaloConfig, build_halo_types(cfg) -> [HaloRegion], run_exchange(cfg,
    profile) -> ExchangeReport, plus device fill/verify helpers and the
    batch (many-jobs-one-launch) API the exchange is built on.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from . import TypeDef, _buffer, _capi, _check, _stream, commit_type
from ._capi import lib

FUSED, COPY, FUSED_ASYNC, DIRECT = 0, 1, 2, 3


@dataclass
class HaloConfig:                  # halo.hpp:25-30
    ranks: tuple = (1, 1, 1)
    interior: tuple = (16, 16, 16)
    radius: int = 3
    element_bytes: int = 64

    def c(self):
        h = _capi.HaloConfig()
        for a in range(3):
            h.ranks[a] = self.ranks[a]
            h.interior[a] = self.interior[a]
        h.radius = self.radius
        h.element_bytes = self.element_bytes
        return h


@dataclass
class HaloRegion:                  # halo.hpp:47-52
    dir: tuple
    send: object                   # CommittedType
    recv: object
    gridpoints: int


@dataclass
class ExchangeReport:              # halo.hpp:132-138 + measured device times
    pack_seconds: float
    alltoallv_seconds: float
    unpack_seconds: float
    verified: bool
    bytes_moved: int
    mismatched_cells: int
    measured_pack_seconds: float
    measured_exchange_seconds: float
    measured_unpack_seconds: float


def build_halo_types(cfg: HaloConfig) -> List[HaloRegion]:
    """halo.hpp:98-130 -- 26 committed (send, recv) region types."""
    send = (_capi.sp_type * 26)()
    recv = (_capi.sp_type * 26)()
    d = (C.c_int * 78)()
    cells = (C.c_int64 * 26)()
    _check(lib.sp_halo_types(C.byref(cfg.c()), send, recv, d, cells))
    out = []
    for k in range(26):
        s = TypeDef(send[k], f"halo.send[{k}]")
        r = TypeDef(recv[k], f"halo.recv[{k}]")
        out.append(HaloRegion((d[3 * k], d[3 * k + 1], d[3 * k + 2]), commit_type(s), commit_type(r), cells[k]))
    return out


def neighbor(cfg: HaloConfig, rank: int, d: Sequence[int]) -> int:
    n = C.c_int64()
    _check(lib.sp_halo_neighbor(C.byref(cfg.c()), rank, (C.c_int * 3)(*d), C.byref(n)))
    return n.value


def fill(cfg: HaloConfig, rank: int, alloc, stream=None):
    a, n, cu = _buffer(alloc, True)
    _check(lib.sp_halo_fill(C.byref(cfg.c()), rank, a, _stream(stream, cu)))


def verify(cfg: HaloConfig, rank: int, alloc, stream=None) -> int:
    """number of padded cells differing from the wrapped global pattern"""
    a, n, cu = _buffer(alloc, False)
    bad = C.c_int64()
    _check(lib.sp_halo_verify(C.byref(cfg.c()), rank, a, _stream(stream, cu), C.byref(bad)))
    return bad.value


def run_exchange(cfg: HaloConfig, profile=None, method: int = FUSED, iters: int = 1) -> ExchangeReport:
    """halo.hpp:172 -- every rank on the current device."""
    rep = _capi.HaloReport()
    _check(lib.sp_halo_run(C.byref(cfg.c()), profile.handle if profile is not None else None,
                           method, iters, C.byref(rep)))
    return ExchangeReport(rep.pack_seconds, rep.alltoallv_seconds, rep.unpack_seconds, bool(rep.verified),
                          rep.bytes_moved, rep.mismatched_cells, rep.measured_pack_seconds,
                          rep.measured_exchange_seconds, rep.measured_unpack_seconds)


class Batch:
    """Persistent many-jobs-one-launch plan (sp_batch_*). jobs: sequence of
    (src, ct, count, dst, position) exactly like pack()/unpack() arguments;
    buffers: CUDA tensors or (address, nbytes)."""

    def __init__(self, jobs, unpack: bool = False):
        arr = (_capi.BatchJob * max(len(jobs), 1))()
        self._keep = []
        for i, (src, ct, count, dst, position) in enumerate(jobs):
            sa, sn, _ = _buffer(src, False)
            da, dn, _ = _buffer(dst, True)
            arr[i] = _capi.BatchJob(sa, sn, ct.handle, count, da, dn, position)
            self._keep.append(ct)
        h = C.c_void_p()
        _check(lib.sp_batch_create(arr, len(jobs), int(unpack), C.byref(h)))
        self.handle = h.value

    @classmethod
    def copies(cls, jobs):
        """Typed copies in one launch (sp_copy_batch_create): jobs are
        (src, src_ct, src_count, dst, dst_ct, dst_count); byte k of the
        source's pack order lands on byte k of the destination's."""
        self = cls.__new__(cls)
        arr = (_capi.CopyJob * max(len(jobs), 1))()
        self._keep = []
        for i, (src, sct, sn_, dst, dct, dn_) in enumerate(jobs):
            sa, sn, _ = _buffer(src, False)
            da, dn, _ = _buffer(dst, True)
            arr[i] = _capi.CopyJob(sa, sn, sct.handle, sn_, da, dn, dct.handle, dn_)
            self._keep += [sct, dct]
        h = C.c_void_p()
        _check(lib.sp_copy_batch_create(arr, len(jobs), C.byref(h)))
        self.handle = h.value
        return self

    def __del__(self):
        try:
            lib.sp_batch_free(self.handle)
        except Exception:
            pass

    def execute(self, stream=None):
        _check(lib.sp_batch_execute(self.handle, _stream(stream, True)))

    @property
    def bytes(self) -> int:
        v = C.c_int64()
        _check(lib.sp_batch_bytes(self.handle, C.byref(v)))
        return v.value
