"""Send-method model over a machine profile (paper Eqs. 1-3), executed by
libstridepack_b200 (csrc/model.cpp). Mirrors the reference's
perf_model.hpp / profile_io.hpp interface:

    MachineProfile, load_profile / load_profile_file / save_profile,
    interp_1d / interp_2d, t_device / t_oneshot / t_staged,
    choose_method(profile, ModelQuery) -> MethodChoice, ModelCache.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass
from typing import Sequence

from . import _capi, _check
from ._capi import lib

CURVES = {"cpu_cpu": 0, "gpu_gpu": 1, "d2h": 2, "h2d": 3}
SURFACES = {"gpu_pack": 0, "gpu_unpack": 1, "host_pack": 2, "host_unpack": 3,
            # B200 extension (optional): the DIRECT method's typed copy, same GPU / peer GPU
            "gpu_direct": 4, "gpu_direct_peer": 5}
DEFAULT_B200_PROFILE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "profiles", "b200.profile")


class MethodChoice(enum.IntEnum):  # perf_model.hpp:46
    OneShot = 0
    Device = 1
    Staged = 2
    Direct = 3                     # B200 extension (choose_method_b200 only)


class Destination(enum.IntEnum):  # where the receive buffer lives (choose_method_b200)
    Host = 0
    SameGpu = 1
    PeerGpu = 2


@dataclass(frozen=True)
class ModelQuery:                  # perf_model.hpp:60-65
    object_size: int
    block_size: int


class MachineProfile:
    """Owns an sp_profile handle (perf_model.hpp:36-45)."""

    def __init__(self, handle=None):
        if handle is None:
            h = C.c_void_p()
            _check(lib.sp_profile_create(C.byref(h)))
            handle = h.value
        self.handle = handle

    def __del__(self):
        try:
            lib.sp_profile_free(self.handle)
        except Exception:
            pass

    def set_curve(self, name: str, sizes: Sequence[float], times: Sequence[float]):
        n = len(sizes)
        arr = C.c_double * max(n, 1)
        _check(lib.sp_profile_set_curve(self.handle, CURVES[name], arr(*sizes), arr(*times), n))

    def set_surface(self, name: str, objects, blocks, times):
        flat = [t for row in times for t in row]
        A = lambda v: (C.c_double * max(len(v), 1))(*v)
        _check(lib.sp_profile_set_surface(self.handle, SURFACES[name], A(objects), len(objects),
                                          A(blocks), len(blocks), A(flat)))


def load_profile(text: str) -> MachineProfile:
    """profile_io.hpp:88 (from text)."""
    h = C.c_void_p()
    _check(lib.sp_profile_parse(text.encode(), C.byref(h)))
    return MachineProfile(h.value)


def load_profile_file(path: str) -> MachineProfile:
    """profile_io.hpp:166"""
    h = C.c_void_p()
    _check(lib.sp_profile_load(os.fsencode(path), C.byref(h)))
    return MachineProfile(h.value)


def save_profile(p: MachineProfile, header: str = "") -> str:
    """profile_io.hpp:174"""
    n = C.c_int64()
    _check(lib.sp_profile_save(p.handle, header.encode(), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(lib.sp_profile_save(p.handle, header.encode(), buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def interp_1d(p: MachineProfile, curve: str, size: float) -> float:
    t = C.c_double()
    _check(lib.sp_interp_1d(p.handle, CURVES[curve], size, C.byref(t)))
    return t.value


def interp_2d(p: MachineProfile, surface: str, obj: float, blk: float) -> float:
    t = C.c_double()
    _check(lib.sp_interp_2d(p.handle, SURFACES[surface], obj, blk, C.byref(t)))
    return t.value


def model_times(p: MachineProfile, q: ModelQuery):
    a, b, c = C.c_double(), C.c_double(), C.c_double()
    _check(lib.sp_model_times(p.handle, q.object_size, q.block_size, C.byref(a), C.byref(b), C.byref(c)))
    return a.value, b.value, c.value


def t_device(p, q):
    return model_times(p, q)[0]


def t_oneshot(p, q):
    return model_times(p, q)[1]


def t_staged(p, q):
    return model_times(p, q)[2]


def choose_method(p: MachineProfile, q: ModelQuery) -> MethodChoice:
    """perf_model.hpp:163"""
    m = C.c_int()
    _check(lib.sp_choose_method(p.handle, q.object_size, q.block_size, C.byref(m)))
    return MethodChoice(m.value)


def choose_method_b200(p: MachineProfile, q: ModelQuery, dst: Destination):
    """B200 extension: Eqs. 1-3 plus Eq. 4 (DIRECT = the measured gpu_direct
    / gpu_direct_peer surface of a device destination). Returns (choice,
    (t_device, t_oneshot, t_staged, t_direct)); t_direct is inf when DIRECT
    is not a candidate."""
    m = C.c_int()
    t = (C.c_double * 4)()
    _check(lib.sp_choose_method_b200(p.handle, q.object_size, q.block_size, int(dst), C.byref(m), t))
    return MethodChoice(m.value), tuple(t)


class ModelCache:
    """perf_model.hpp:184-229 -- memoised choose_method, safe for concurrent
    readers; keeps its own reference to the profile."""

    def __init__(self, p: MachineProfile):
        h = C.c_void_p()
        _check(lib.sp_model_cache_create(p.handle, C.byref(h)))
        self.handle = h.value
        self.profile = p

    def __del__(self):
        try:
            lib.sp_model_cache_free(self.handle)
        except Exception:
            pass

    def choose(self, q: ModelQuery) -> MethodChoice:
        m = C.c_int()
        _check(lib.sp_model_cache_choose(self.handle, q.object_size, q.block_size, C.byref(m)))
        return MethodChoice(m.value)
