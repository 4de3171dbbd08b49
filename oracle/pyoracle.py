"""oracle/pyoracle.py -- TEST INFRASTRUCTURE ONLY.

ctypes bindings for the two CPU checkers:

* ``Oracle``    -- oracle/liboracle.so, our plain-C restatement (oracle.c) of
  the reference algorithm (commit + pack/unpack), and
* ``Reference`` -- oracle/_ref/libstridepack_ref.so, the UNMODIFIED reference
  headers compiled in place by oracle/Makefile (present whenever this repo
  was built in a container that had /root/reference; it travels with the
  snapshot).

Only tests/, bench.py (cpu_baseline / --impl reference) and
__graft_entry__.smoke() import this module, and only as the checker: the
product library (paper_2012_14363_b200) never loads either .so.

Type programs: flat int64 prefix encoding, see oracle/ref_harness.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libstridepack_ref.so")
MAXD = 64

# status codes: proj/include/stridepack/errors.hpp:8-47
OK, INVALID_ARGUMENT, UNSUPPORTED_ORDER, INVALID_LAYOUT = 0, 1, 2, 3
BUFFER_TOO_SMALL, OVERLAPPING_LAYOUT, UNSUPPORTED = 4, 5, 6
EMPTY_PROFILE, PARSE_ERROR, OTHER, BAD_PROGRAM = 7, 8, 9, 10

i64p = C.POINTER(C.c_int64)
u8p = C.POINTER(C.c_uint8)


class CommitInfo(C.Structure):
    _fields_ = [
        ("form", C.c_int64), ("size", C.c_int64), ("extent", C.c_int64),
        ("span", C.c_int64), ("overlapping", C.c_int64), ("ndims", C.c_int64),
        ("start", C.c_int64), ("counts", C.c_int64 * MAXD),
        ("strides", C.c_int64 * MAXD), ("word", C.c_int64),
        ("block", C.c_int64 * 3), ("grid", C.c_int64 * 3),
        ("strategy", C.c_int64), ("n_fallback_runs", C.c_int64),
        ("simplify_rounds", C.c_int64),
    ]


@dataclass
class Commit:
    """Mirror of commit.hpp:30-43 (CommittedType) minus the definition."""
    status: int
    form: int = 0            # 0 Strided, 1 Empty, 2 Unsupported
    size: int = 0
    extent: int = 0
    span: int = 0
    overlapping: bool = False
    start: int = 0
    counts: list = field(default_factory=list)
    strides: list = field(default_factory=list)
    word: int = 0
    block: tuple = ()
    grid: tuple = ()
    strategy: int = 0        # 0 gridz, 1 iterate
    n_fallback_runs: int = 0
    simplify_rounds: int = -1

    def canon(self):
        if self.form != 0:
            return None
        return (self.start, tuple(self.counts), tuple(self.strides))

    def plan(self):
        if self.form != 0:
            return None
        return (self.word, self.block, self.grid, self.strategy)


def _arr(prog):
    a = np.ascontiguousarray(np.asarray(prog, dtype=np.int64))
    return a, a.ctypes.data_as(i64p), len(a)


def _buf(b):
    """numpy uint8 view (contiguous) + pointer."""
    a = np.ascontiguousarray(b, dtype=np.uint8)
    return a, a.ctypes.data_as(u8p)


class _Engine:
    prefix = ""

    def __init__(self, path):
        self.path = path
        self.lib = C.CDLL(path)
        p = self.prefix
        f = getattr(self.lib, p + "commit")
        f.argtypes = [i64p, C.c_int64, C.POINTER(CommitInfo)]
        f.restype = C.c_int
        f = getattr(self.lib, p + "size_extent")
        f.argtypes = [i64p, C.c_int64, i64p, i64p]
        f.restype = C.c_int
        f = getattr(self.lib, p + "flatten")
        f.argtypes = [i64p, C.c_int64, i64p, i64p, C.c_int64, i64p, i64p]
        f.restype = C.c_int
        f = getattr(self.lib, p + "commit_handle")
        f.argtypes = [i64p, C.c_int64, C.POINTER(C.c_int)]
        f.restype = C.c_void_p
        f = getattr(self.lib, p + "free_handle")
        f.argtypes = [C.c_void_p]
        f.restype = None

    # -- commit -----------------------------------------------------------
    def commit(self, prog) -> Commit:
        a, ptr, n = _arr(prog)
        info = CommitInfo()
        st = getattr(self.lib, self.prefix + "commit")(ptr, n, C.byref(info))
        if st != OK:
            return Commit(status=st)
        nd = info.ndims
        return Commit(
            status=OK, form=info.form, size=info.size, extent=info.extent,
            span=info.span, overlapping=bool(info.overlapping),
            start=info.start, counts=list(info.counts[:nd]),
            strides=list(info.strides[:nd]), word=info.word,
            block=tuple(info.block), grid=tuple(info.grid),
            strategy=info.strategy, n_fallback_runs=info.n_fallback_runs,
            simplify_rounds=info.simplify_rounds)

    def size_extent(self, prog):
        a, ptr, n = _arr(prog)
        s, e = C.c_int64(), C.c_int64()
        st = getattr(self.lib, self.prefix + "size_extent")(ptr, n, C.byref(s), C.byref(e))
        return st, s.value, e.value

    def flatten(self, prog):
        """normalized block list + overlap flag (block_list.hpp:129)."""
        a, ptr, n = _arr(prog)
        cnt, ov = C.c_int64(), C.c_int64()
        fn = getattr(self.lib, self.prefix + "flatten")
        st = fn(ptr, n, None, None, 0, C.byref(cnt), C.byref(ov))
        if st != OK:
            return st, None, None
        offs = np.zeros(max(cnt.value, 1), np.int64)
        lens = np.zeros(max(cnt.value, 1), np.int64)
        st = fn(ptr, n, offs.ctypes.data_as(i64p), lens.ctypes.data_as(i64p),
                cnt.value, C.byref(cnt), C.byref(ov))
        return st, list(zip(offs[:cnt.value].tolist(), lens[:cnt.value].tolist())), bool(ov.value)

    # -- pack / unpack ------------------------------------------------------
    def handle(self, prog):
        a, ptr, n = _arr(prog)
        st = C.c_int()
        h = getattr(self.lib, self.prefix + "commit_handle")(ptr, n, C.byref(st))
        if not h:
            raise RuntimeError(f"commit failed with status {st.value}")
        return Handle(self, h)


class Handle:
    def __init__(self, eng, h):
        self.eng, self.h = eng, h

    def __del__(self):
        try:
            getattr(self.eng.lib, self.eng.prefix + "free_handle")(self.h)
        except Exception:
            pass


class Oracle(_Engine):
    """oracle/oracle.c -- the C restatement."""
    prefix = "or_"

    def __init__(self, path=ORACLE_SO):
        super().__init__(path)
        L = self.lib
        L.or_pack.argtypes = [i64p, C.c_int64, u8p, C.c_uint64, C.c_int64, u8p,
                              C.c_uint64, C.c_int64, C.c_int, i64p]
        L.or_unpack.argtypes = [i64p, C.c_int64, u8p, C.c_uint64, C.c_int64,
                                C.c_int64, u8p, C.c_uint64, C.c_int, i64p]
        L.or_pack_h.argtypes = [C.c_void_p, u8p, C.c_uint64, C.c_int64, u8p,
                                C.c_uint64, C.c_int64, i64p]
        L.or_unpack_h.argtypes = [C.c_void_p, u8p, C.c_uint64, C.c_int64,
                                  C.c_int64, u8p, C.c_uint64, i64p]

    def pack(self, prog, src, incount, dst, position=0, allow_fallback=True):
        """returns (status, new_position); dst (np.uint8) is written in place."""
        a, ptr, n = _arr(prog)
        s, sp = _buf(src)
        assert dst.flags.c_contiguous and dst.dtype == np.uint8
        npos = C.c_int64()
        st = self.lib.or_pack(ptr, n, sp, s.nbytes, incount,
                              dst.ctypes.data_as(u8p), dst.nbytes, position,
                              int(allow_fallback), C.byref(npos))
        return st, npos.value

    def unpack(self, prog, src, position, outcount, dst, allow_fallback=True):
        a, ptr, n = _arr(prog)
        s, sp = _buf(src)
        assert dst.flags.c_contiguous and dst.dtype == np.uint8
        npos = C.c_int64()
        st = self.lib.or_unpack(ptr, n, sp, s.nbytes, position, outcount,
                                dst.ctypes.data_as(u8p), dst.nbytes,
                                int(allow_fallback), C.byref(npos))
        return st, npos.value

    def pack_h(self, h, src_ptr, src_len, incount, dst_ptr, dst_len, position=0):
        npos = C.c_int64()
        st = self.lib.or_pack_h(h.h, C.cast(src_ptr, u8p), src_len, incount,
                                C.cast(dst_ptr, u8p), dst_len, position, C.byref(npos))
        return st, npos.value

    def unpack_h(self, h, src_ptr, src_len, position, outcount, dst_ptr, dst_len):
        npos = C.c_int64()
        st = self.lib.or_unpack_h(h.h, C.cast(src_ptr, u8p), src_len, position,
                                  outcount, C.cast(dst_ptr, u8p), dst_len, C.byref(npos))
        return st, npos.value


class Reference(_Engine):
    """oracle/_ref/libstridepack_ref.so -- the reference, compiled in place."""
    prefix = "ref_"

    def __init__(self, path=REF_SO):
        super().__init__(path)
        L = self.lib
        L.ref_pack.argtypes = [i64p, C.c_int64, u8p, C.c_uint64, C.c_int64, u8p,
                               C.c_uint64, C.c_int64, C.c_int, C.c_int, i64p]
        L.ref_unpack.argtypes = [i64p, C.c_int64, u8p, C.c_uint64, C.c_int64,
                                 C.c_int64, u8p, C.c_uint64, C.c_int, C.c_int, i64p]
        L.ref_pack_h.argtypes = [C.c_void_p, u8p, C.c_uint64, C.c_int64, u8p,
                                 C.c_uint64, C.c_int64, C.c_int, i64p]
        L.ref_unpack_h.argtypes = [C.c_void_p, u8p, C.c_uint64, C.c_int64,
                                   C.c_int64, u8p, C.c_uint64, C.c_int, i64p]
        L.ref_corpus.argtypes = [C.c_uint64, C.c_int64, C.c_int, i64p, C.c_int64]
        L.ref_corpus.restype = C.c_int64
        L.ref_profile_load.argtypes = [C.c_char_p, C.POINTER(C.c_int)]
        L.ref_profile_load.restype = C.c_void_p
        L.ref_profile_parse.argtypes = [C.c_char_p, C.POINTER(C.c_int)]
        L.ref_profile_parse.restype = C.c_void_p
        L.ref_profile_free.argtypes = [C.c_void_p]
        L.ref_profile_save.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_int64]
        L.ref_profile_save.restype = C.c_int64
        L.ref_profile_scaled.argtypes = [C.c_void_p, C.c_double]
        L.ref_profile_scaled.restype = C.c_void_p
        L.ref_choose.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.POINTER(C.c_int),
                                 C.POINTER(C.c_double), C.POINTER(C.c_double),
                                 C.POINTER(C.c_double)]
        L.ref_run_exchange.argtypes = [i64p, i64p, C.c_int64, C.c_int64, C.c_void_p,
                                       C.c_void_p]
        L.ref_halo_types.argtypes = [i64p, C.c_int64, C.c_int64, i64p, C.c_int64]
        L.ref_halo_types.restype = C.c_int64
        L.ref_fill_cell.argtypes = [u8p, C.c_int64, C.c_int64, C.c_int64, C.c_int64]

    def pack(self, prog, src, incount, dst, position=0, threads=1, allow_fallback=True):
        a, ptr, n = _arr(prog)
        s, sp = _buf(src)
        npos = C.c_int64()
        st = self.lib.ref_pack(ptr, n, sp, s.nbytes, incount,
                               dst.ctypes.data_as(u8p), dst.nbytes, position,
                               threads, int(allow_fallback), C.byref(npos))
        return st, npos.value

    def unpack(self, prog, src, position, outcount, dst, threads=1, allow_fallback=True):
        a, ptr, n = _arr(prog)
        s, sp = _buf(src)
        npos = C.c_int64()
        st = self.lib.ref_unpack(ptr, n, sp, s.nbytes, position, outcount,
                                 dst.ctypes.data_as(u8p), dst.nbytes, threads,
                                 int(allow_fallback), C.byref(npos))
        return st, npos.value

    def pack_h(self, h, src_ptr, src_len, incount, dst_ptr, dst_len, position=0, threads=1):
        npos = C.c_int64()
        st = self.lib.ref_pack_h(h.h, C.cast(src_ptr, u8p), src_len, incount,
                                 C.cast(dst_ptr, u8p), dst_len, position, threads,
                                 C.byref(npos))
        return st, npos.value

    def unpack_h(self, h, src_ptr, src_len, position, outcount, dst_ptr, dst_len, threads=1):
        npos = C.c_int64()
        st = self.lib.ref_unpack_h(h.h, C.cast(src_ptr, u8p), src_len, position,
                                   outcount, C.cast(dst_ptr, u8p), dst_len, threads,
                                   C.byref(npos))
        return st, npos.value

    def corpus(self, seed, count, mode):
        """the reference generator (tests/test_util.hpp:86-151) -> programs."""
        need = self.lib.ref_corpus(seed, count, mode, None, 0)
        buf = np.zeros(-need, np.int64)
        got = self.lib.ref_corpus(seed, count, mode, buf.ctypes.data_as(i64p), len(buf))
        assert got == -need
        out, at = [], 0
        while at < got:
            ln = int(buf[at])
            out.append(buf[at + 1: at + 1 + ln].tolist())
            at += 1 + ln
        return out


def split_programs(buf):
    out, at = [], 0
    while at < len(buf):
        ln = int(buf[at])
        out.append(list(buf[at + 1: at + 1 + ln]))
        at += 1 + ln
    return out


_oracle = None
_ref = None


def oracle() -> Oracle:
    global _oracle
    if _oracle is None:
        _oracle = Oracle()
    return _oracle


def reference():
    """The compiled reference, or None when oracle/_ref was never built."""
    global _ref
    if _ref is None and os.path.exists(REF_SO):
        _ref = Reference()
    return _ref
