"""paper_2012_14363_b200 -- B200-native engine for non-contiguous MPI datatypes.

Python mirror of the reference engine's interface ("stridepack",
/root/reference/proj/include/stridepack/), executed by
libstridepack_b200.so: the datatype pipeline runs in C++ and every
pack/unpack runs as an sm_100a kernel. Names, argument meaning and error
behaviour follow the reference so its tests read the same here:

    make_named / make_contiguous / make_vector / make_hvector /
    make_subarray                      type_def.hpp:125-195
    type_size / type_extent            type_def.hpp:198-250
    commit_type -> CommittedType       commit.hpp:51-79
    pack / unpack                      pack.hpp:99 / :143
    exceptions                         errors.hpp:8-47

Buffers may be CUDA tensors (device or pinned host), numpy arrays / bytearrays
(pageable host: staged through the device) or ``(address, nbytes)`` tuples.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import Optional, Sequence

from . import _capi
from ._capi import lib

__all__ = [
    "Error", "InvalidArgument", "UnsupportedOrder", "InvalidLayout", "BufferTooSmall",
    "OverlappingLayout", "Unsupported", "EmptyProfile", "ParseError", "CudaError",
    "NoDevice", "InvalidHandle", "InternalError",
    "NamedKind", "ArrayOrder", "CanonForm", "CountStrategy", "Kernel",
    "TypeDef", "make_named", "make_contiguous", "make_vector", "make_hvector",
    "make_subarray", "make_indexed", "make_hindexed", "make_indexed_block", "make_hindexed_block",
    "make_struct", "make_resized", "type_size", "type_extent", "from_program",
    "StridedBlock", "PackPlan", "CommittedType", "commit_type", "pack", "unpack",
    "last_launch", "kernel_launch_count",
]


# ------------------------------------------------------------------ errors
class Error(RuntimeError):
    """errors.hpp:8 -- base of every engine error."""


class InvalidArgument(Error):
    pass


class UnsupportedOrder(Error):
    pass


class InvalidLayout(Error):
    pass


class BufferTooSmall(Error):
    pass


class OverlappingLayout(Error):
    pass


class Unsupported(Error):
    pass


class EmptyProfile(Error):
    pass


class ParseError(Error):
    pass


class InternalError(Error):
    pass


class InvalidHandle(Error):
    pass


class CudaError(Error):
    pass


class NoDevice(Error):
    pass


class Timeout(Error):
    """a peer rank exited, or did not answer within TEMPI_TIMEOUT seconds"""


_ERRORS = {1: InvalidArgument, 2: UnsupportedOrder, 3: InvalidLayout, 4: BufferTooSmall,
           5: OverlappingLayout, 6: Unsupported, 7: EmptyProfile, 8: ParseError,
           9: InternalError, 11: InvalidHandle, 12: CudaError, 13: NoDevice, 14: Timeout}


def _check(status: int) -> None:
    if status != 0:
        msg = lib.sp_last_error().decode() or lib.sp_status_string(status).decode()
        raise _ERRORS.get(status, Error)(msg)


# ------------------------------------------------------------------ enums
class NamedKind(enum.IntEnum):   # type_def.hpp:15
    Byte = 0
    Int = 1
    Float = 2
    Double = 3


class ArrayOrder(enum.IntEnum):  # type_def.hpp:47
    C = 0
    Fortran = 1


class CanonForm(enum.IntEnum):   # commit.hpp:21-25
    Strided = 0
    Empty = 1
    Unsupported = 2


class CountStrategy(enum.IntEnum):  # plan.hpp:13-16
    GridZ = 0
    Iterate = 1


class Kernel(enum.IntEnum):
    Auto = 0
    Words = 1
    SmallRow = 2
    BlockList = 3
    TMA = 4
    Words64 = 5
    Batch = 6
    Shift = 7
    DMA = 8


# ------------------------------------------------------------------ types
class TypeDef:
    """A datatype definition handle (type_def.hpp:52-123)."""

    __slots__ = ("handle", "_committed", "_desc")

    def __init__(self, handle: int, desc: str):
        self.handle = handle
        self._committed = None
        self._desc = desc

    def __del__(self):
        try:
            lib.sp_type_free(self.handle)
        except Exception:
            pass

    def size(self) -> int:
        v = C.c_int64()
        _check(lib.sp_type_size(self.handle, C.byref(v)))
        return v.value

    def extent(self) -> int:
        v = C.c_int64()
        _check(lib.sp_type_extent(self.handle, C.byref(v)))
        return v.value

    def lb(self) -> int:
        """MPI lower bound (0 for every reference constructor)"""
        v = C.c_int64()
        _check(lib.sp_type_lb(self.handle, C.byref(v)))
        return v.value

    def str(self) -> str:
        return self._desc

    __str__ = str

    def __repr__(self):
        return f"TypeDef({self._desc})"


def _new(fn, *args, desc) -> TypeDef:
    h = _capi.sp_type()
    _check(fn(*args, C.byref(h)))
    return TypeDef(h.value, desc)


_NAMES = {0: "byte", 1: "int", 2: "float", 3: "double"}


def make_named(kind: NamedKind) -> TypeDef:
    return _new(lib.sp_type_named, int(kind), desc=_NAMES.get(int(kind), "?"))


def make_contiguous(count: int, inner: TypeDef) -> TypeDef:
    return _new(lib.sp_type_contiguous, count, inner.handle, desc=f"contiguous({count},{inner})")


def make_vector(count: int, blocklength: int, stride: int, inner: TypeDef) -> TypeDef:
    return _new(lib.sp_type_vector, count, blocklength, stride, inner.handle,
                desc=f"vector({count},{blocklength},{stride},{inner})")


def make_hvector(count: int, blocklength: int, stride_bytes: int, inner: TypeDef) -> TypeDef:
    return _new(lib.sp_type_hvector, count, blocklength, stride_bytes, inner.handle,
                desc=f"hvector({count},{blocklength},{stride_bytes},{inner})")


def make_subarray(ndims: int, sizes: Sequence[int], subsizes: Sequence[int],
                  offsets: Sequence[int], inner: TypeDef,
                  order: ArrayOrder = ArrayOrder.C) -> TypeDef:
    n = max(len(sizes), len(subsizes), len(offsets), 1)
    if len(sizes) != ndims or len(subsizes) != ndims or len(offsets) != ndims:
        raise InvalidArgument("subarray: sizes/subsizes/offsets must have ndims entries")
    arr = C.c_int64 * n
    lst = lambda v: "[" + ",".join(str(x) for x in v) + "]"
    return _new(lib.sp_type_subarray, ndims, arr(*sizes), arr(*subsizes), arr(*offsets),
                inner.handle, int(order),
                desc=f"subarray({ndims},{lst(sizes)},{lst(subsizes)},{lst(offsets)},{inner})")


# ---- beyond the reference (MPI-3.1 4.1.2-4.1.7; PAPER.md:1164 future work)
def _arr(v):
    return (C.c_int64 * max(len(v), 1))(*[int(x) for x in v])


def _lst(v):
    return "[" + ",".join(str(int(x)) for x in v) + "]"


def make_indexed(blocklengths: Sequence[int], displacements: Sequence[int], inner: TypeDef) -> TypeDef:
    """MPI_Type_indexed: displacements in inner extents"""
    if len(blocklengths) != len(displacements):
        raise InvalidArgument("indexed: one displacement per block")
    return _new(lib.sp_type_indexed, len(blocklengths), _arr(blocklengths), _arr(displacements), inner.handle,
                desc=f"indexed({_lst(blocklengths)},{_lst(displacements)},{inner})")


def make_hindexed(blocklengths: Sequence[int], displacements: Sequence[int], inner: TypeDef) -> TypeDef:
    """MPI_Type_create_hindexed: displacements in bytes"""
    if len(blocklengths) != len(displacements):
        raise InvalidArgument("hindexed: one displacement per block")
    return _new(lib.sp_type_hindexed, len(blocklengths), _arr(blocklengths), _arr(displacements), inner.handle,
                desc=f"hindexed({_lst(blocklengths)},{_lst(displacements)},{inner})")


def make_indexed_block(blocklength: int, displacements: Sequence[int], inner: TypeDef) -> TypeDef:
    """MPI_Type_create_indexed_block"""
    return _new(lib.sp_type_indexed_block, len(displacements), blocklength, _arr(displacements), inner.handle,
                desc=f"indexed_block({blocklength},{_lst(displacements)},{inner})")


def make_hindexed_block(blocklength: int, displacements: Sequence[int], inner: TypeDef) -> TypeDef:
    """MPI_Type_create_hindexed_block"""
    return _new(lib.sp_type_hindexed_block, len(displacements), blocklength, _arr(displacements), inner.handle,
                desc=f"hindexed_block({blocklength},{_lst(displacements)},{inner})")


def make_struct(blocklengths: Sequence[int], displacements: Sequence[int], types: Sequence[TypeDef]) -> TypeDef:
    """MPI_Type_create_struct: displacements in bytes, one type per block"""
    if not (len(blocklengths) == len(displacements) == len(types)):
        raise InvalidArgument("struct: one displacement and one type per block")
    th = (_capi.sp_type * max(len(types), 1))(*[t.handle for t in types])
    return _new(lib.sp_type_struct, len(types), _arr(blocklengths), _arr(displacements), th,
                desc=f"struct({_lst(blocklengths)},{_lst(displacements)},[{','.join(str(t) for t in types)}])")


def make_resized(inner: TypeDef, lb: int, extent: int) -> TypeDef:
    """MPI_Type_create_resized"""
    return _new(lib.sp_type_resized, inner.handle, lb, extent, desc=f"resized({inner},{lb},{extent})")


@dataclass(frozen=True)
class Block:                       # block_list.hpp:13-18
    offset: int
    length: int


@dataclass(frozen=True)
class BlockList:                   # block_list.hpp:20-40
    blocks: tuple
    overlap: bool

    def total_length(self) -> int:
        return sum(b.length for b in self.blocks)

    def span(self) -> int:
        return self.blocks[-1].offset + self.blocks[-1].length if self.blocks else 0


def flatten(d: TypeDef) -> BlockList:
    """The definition's normalized byte runs (flatten_oracle,
    block_list.hpp:123-126; the CLI's `flatten`)."""
    n = C.c_int64()
    ov = C.c_int()
    _check(lib.sp_type_flatten(d.handle, None, None, 0, C.byref(n), C.byref(ov)))
    off = (C.c_int64 * max(n.value, 1))()
    ln = (C.c_int64 * max(n.value, 1))()
    _check(lib.sp_type_flatten(d.handle, off, ln, n.value, C.byref(n), C.byref(ov)))
    return BlockList(tuple(Block(off[i], ln[i]) for i in range(n.value)), bool(ov.value))


# the reference's name for the same list (block_list.hpp:123-126)
flatten_oracle = flatten


def normalize_blocks(runs) -> BlockList:
    """block_list.hpp:44-61: drop empty runs, sort by (offset, length),
    merge abutting / overlapping runs; overlap = some byte described twice.
    runs: iterable of (offset, length) or Block."""
    rs = sorted(((r.offset, r.length) if isinstance(r, Block) else (int(r[0]), int(r[1])))
                for r in runs)
    out, overlap = [], False
    for off, ln in rs:
        if ln == 0:
            continue
        if out and off <= out[-1][0] + out[-1][1]:
            if off < out[-1][0] + out[-1][1]:
                overlap = True
            end = max(out[-1][0] + out[-1][1], off + ln)
            out[-1] = (out[-1][0], end - out[-1][0])
        else:
            out.append((off, ln))
    return BlockList(tuple(Block(o, l) for o, l in out), overlap)


def enumerate_blocks(sb: "StridedBlock") -> BlockList:
    """block_list.hpp:129-159: the normalized runs a StridedBlock describes
    (counts[0] bytes per run, dimension 1 fastest)."""
    if any(c < 1 for c in sb.counts):
        return BlockList((), False)
    import itertools
    runs = []
    dims = [range(c) for c in sb.counts[1:]]
    for idx in itertools.product(*reversed(dims)):
        off = sb.start + sum(i * st for i, st in zip(reversed(idx), sb.strides[1:]))
        runs.append((off, sb.counts[0]))
    return normalize_blocks(runs)


@dataclass(frozen=True)
class TypeFileResult:              # typefile.hpp:27-30
    name: str
    def_: TypeDef


def parse_type_file(text: str) -> TypeFileResult:
    """typefile.hpp:131-258: `type <name> = <ctor>(...)` lines and one final
    `commit <name>`; errors raise ParseError("line N: ...")."""
    h = _capi.sp_type()
    name = C.create_string_buffer(256)
    _check(lib.sp_typefile_parse(text.encode(), C.byref(h), name, 256))
    nm = name.value.decode()
    return TypeFileResult(nm, TypeDef(h.value, f"typefile:{nm}"))


def type_size(d: TypeDef) -> int:
    return d.size()


def type_extent(d: TypeDef) -> int:
    return d.extent()


def from_program(prog: Sequence[int]) -> TypeDef:
    """Build a definition from the flat int64 type program used by the
    checkers (layout documented in oracle/ref_harness.cpp)."""
    prog = [int(x) for x in prog]
    at = 0

    def nxt():
        nonlocal at
        if at >= len(prog):
            raise InvalidArgument("truncated type program")
        v = prog[at]
        at += 1
        return v

    def rec():
        tag = nxt()
        if tag == 0:
            return make_named(NamedKind(nxt()))
        if tag == 1:
            c = nxt()
            return make_contiguous(c, rec())
        if tag in (2, 3):
            c, l, s = nxt(), nxt(), nxt()
            inner = rec()
            return (make_vector if tag == 2 else make_hvector)(c, l, s, inner)
        if tag == 4:
            nd, order = nxt(), nxt()
            sz = [nxt() for _ in range(nd)]
            sub = [nxt() for _ in range(nd)]
            off = [nxt() for _ in range(nd)]
            inner = rec()
            return make_subarray(nd, sz, sub, off, inner, ArrayOrder(order))
        raise InvalidArgument(f"bad type program tag {tag}")

    d = rec()
    if at != len(prog):
        raise InvalidArgument("trailing type program entries")
    return d


# ------------------------------------------------------------------ commit
@dataclass(frozen=True)
class StridedBlock:                # strided_block.hpp:17-46
    start: int
    counts: tuple
    strides: tuple

    def ndims(self) -> int:
        return len(self.counts)

    def byte_count(self) -> int:
        n = 1
        for c in self.counts:
            n *= c
        return n


@dataclass(frozen=True)
class PackPlan:                    # plan.hpp:27-44
    word: int
    block_dims: tuple
    grid_dims: tuple
    count_strategy: CountStrategy


@dataclass
class CommittedType:               # commit.hpp:30-43
    definition: TypeDef
    form: CanonForm
    canon: Optional[StridedBlock]
    plan: Optional[PackPlan]
    size: int
    extent: int
    span: int
    overlapping: bool
    n_fallback_runs: int
    simplify_rounds: int

    @property
    def handle(self) -> int:
        return self.definition.handle


def commit_type(d: TypeDef) -> CommittedType:
    """commit.hpp:51 -- commits the handle in place (MPI_Type_commit)."""
    _check(lib.sp_type_commit(d.handle))
    info = _capi.TypeInfo()
    cap = 64
    counts = (C.c_int64 * cap)()
    strides = (C.c_int64 * cap)()
    _check(lib.sp_type_query(d.handle, C.byref(info), counts, strides, cap))
    if info.ndims > cap:
        counts = (C.c_int64 * info.ndims)()
        strides = (C.c_int64 * info.ndims)()
        _check(lib.sp_type_query(d.handle, C.byref(info), counts, strides, info.ndims))
    form = CanonForm(info.form)
    canon = plan = None
    if form == CanonForm.Strided:
        nd = info.ndims
        canon = StridedBlock(info.start, tuple(counts[:nd]), tuple(strides[:nd]))
        plan = PackPlan(info.word, tuple(info.block), tuple(info.grid), CountStrategy(info.strategy))
    return CommittedType(d, form, canon, plan, info.size, info.extent, info.span,
                         bool(info.overlapping), info.n_fallback_runs, info.simplify_rounds)


# ------------------------------------------------------------------ buffers
def _buffer(obj, writable: bool):
    """(address, nbytes, is_cuda_tensor) for a supported buffer object."""
    if isinstance(obj, tuple) and len(obj) == 2:
        return int(obj[0]), int(obj[1]), False
    mod = type(obj).__module__
    if mod.startswith("torch"):
        if not obj.is_contiguous():
            raise InvalidArgument("tensor buffers must be contiguous")
        return obj.data_ptr(), obj.numel() * obj.element_size(), obj.is_cuda
    if mod.startswith("numpy"):
        if not obj.flags.c_contiguous:
            raise InvalidArgument("numpy buffers must be C-contiguous")
        if writable and not obj.flags.writeable:
            raise InvalidArgument("destination array is read-only")
        return obj.ctypes.data, obj.nbytes, False
    if isinstance(obj, (bytearray, memoryview)):
        mv = memoryview(obj)
        buf = (C.c_char * mv.nbytes).from_buffer(mv)
        return C.addressof(buf), mv.nbytes, False
    if isinstance(obj, bytes):
        if writable:
            raise InvalidArgument("bytes objects are read-only")
        return C.cast(C.c_char_p(obj), C.c_void_p).value, len(obj), False
    raise InvalidArgument(f"unsupported buffer type {type(obj)!r}")


def _stream(stream, any_cuda: bool):
    if stream is not None:
        return stream if isinstance(stream, int) else int(stream.cuda_stream)
    if any_cuda:
        import torch
        return int(torch.cuda.current_stream().cuda_stream)
    return 0


def _opts(allow_fallback, kernel, force_word):
    return _capi.PackOptions(int(bool(allow_fallback)), int(kernel), int(force_word))


def pack(src, ct: CommittedType, incount: int, dst, position: int = 0, *,
         allow_fallback: bool = True, kernel: Kernel = Kernel.Auto, force_word: int = 0,
         stream=None, sync: bool = False) -> int:
    """pack.hpp:99 -- gather ``incount`` objects of ``ct`` from src into dst at
    ``position``; returns the advanced position. Runs as an sm_100a kernel on
    the current device, ordered on ``stream`` (default: torch's current
    stream when a CUDA tensor is involved, else the legacy stream)."""
    sa, sn, sc = _buffer(src, False)
    da, dn, dc = _buffer(dst, True)
    pos = C.c_int64(position)
    s = _stream(stream, sc or dc)
    o = _opts(allow_fallback, kernel, force_word)
    _check(lib.sp_pack_ex(sa, sn, ct.handle, incount, da, dn, C.byref(pos), s, C.byref(o)))
    if sync:
        _sync(s)
    return pos.value


def unpack(src, position: int, ct: CommittedType, outcount: int, dst, *,
           allow_fallback: bool = True, kernel: Kernel = Kernel.Auto, force_word: int = 0,
           stream=None, sync: bool = False) -> int:
    """pack.hpp:143 -- scatter inverse of pack; bytes of dst outside the
    layout are never written; overlapping layouts are refused."""
    sa, sn, sc = _buffer(src, False)
    da, dn, dc = _buffer(dst, True)
    pos = C.c_int64(position)
    s = _stream(stream, sc or dc)
    o = _opts(allow_fallback, kernel, force_word)
    _check(lib.sp_unpack_ex(sa, sn, C.byref(pos), ct.handle, outcount, da, dn, s, C.byref(o)))
    if sync:
        _sync(s)
    return pos.value


def copy(src, src_ct: CommittedType, src_count: int, dst, dst_ct: CommittedType, dst_count: int, *,
         stream=None, sync: bool = False) -> None:
    """Typed copy (sp_copy): byte k of src_count objects of src_ct in pack
    order lands on byte k of dst_count objects of dst_ct in unpack order --
    pack.hpp:99 fused with pack.hpp:143, one kernel, no packed buffer."""
    sa, sn, sc = _buffer(src, False)
    da, dn, dc = _buffer(dst, True)
    job = _capi.CopyJob(sa, sn, src_ct.handle, src_count, da, dn, dst_ct.handle, dst_count)
    s = _stream(stream, sc or dc)
    _check(lib.sp_copy(C.byref(job), s))
    if sync:
        _sync(s)


def _sync(stream_handle: int):
    import torch
    if stream_handle:
        torch.cuda.ExternalStream(stream_handle).synchronize()
    else:
        torch.cuda.synchronize()


@dataclass
class LaunchInfo:
    kernel: Kernel
    word: int
    launches: int
    grid: int
    block: int
    staged: bool


def last_launch() -> LaunchInfo:
    li = _capi.LaunchInfo()
    _check(lib.sp_last_launch(C.byref(li)))
    return LaunchInfo(Kernel(li.kernel), li.word, li.launches, li.grid, li.block, bool(li.staged))


def kernel_launch_count() -> int:
    return int(lib.sp_kernel_launch_count())
