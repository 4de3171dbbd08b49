"""ctypes binding of include/stridepack_b200.h (libstridepack_b200.so).

The shared library is built in-tree by ``__graft_entry__.build()``
(paper_2012_14363_b200/csrc/Makefile). Importing this module without it
fails loudly: there is no Python or CPU fallback for the datatype engine.
"""
from __future__ import annotations

import ctypes as C
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# SPB_LIB selects another build of the same library (e.g. the ASan/UBSan
# build of `make -C paper_2012_14363_b200/csrc asan`); default: in-tree
LIB_PATH = os.environ.get("SPB_LIB") or os.path.join(PKG_DIR, "libstridepack_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(the B200 engine has no fallback implementation)")

lib = C.CDLL(LIB_PATH)

i64 = C.c_int64
u64 = C.c_uint64
i64p = C.POINTER(C.c_int64)
sp_type = C.c_uint64


class TypeInfo(C.Structure):
    _fields_ = [("form", i64), ("size", i64), ("extent", i64), ("span", i64),
                ("overlapping", i64), ("ndims", i64), ("start", i64), ("word", i64),
                ("block", i64 * 3), ("grid", i64 * 3), ("strategy", i64),
                ("n_fallback_runs", i64), ("simplify_rounds", i64)]


class PackOptions(C.Structure):
    _fields_ = [("allow_fallback", C.c_int), ("kernel", C.c_int), ("force_word", C.c_int)]


class LaunchInfo(C.Structure):
    _fields_ = [("kernel", i64), ("word", i64), ("launches", i64), ("grid", i64),
                ("block", i64), ("staged", i64)]


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("sp_status_string", C.c_char_p, C.c_int)
_sig("sp_last_error", C.c_char_p)
_sig("sp_type_named", C.c_int, C.c_int, C.POINTER(sp_type))
_sig("sp_type_contiguous", C.c_int, i64, sp_type, C.POINTER(sp_type))
_sig("sp_type_vector", C.c_int, i64, i64, i64, sp_type, C.POINTER(sp_type))
_sig("sp_type_hvector", C.c_int, i64, i64, i64, sp_type, C.POINTER(sp_type))
_sig("sp_type_subarray", C.c_int, i64, i64p, i64p, i64p, sp_type, C.c_int, C.POINTER(sp_type))
_sig("sp_type_indexed", C.c_int, i64, i64p, i64p, sp_type, C.POINTER(sp_type))
_sig("sp_type_hindexed", C.c_int, i64, i64p, i64p, sp_type, C.POINTER(sp_type))
_sig("sp_type_indexed_block", C.c_int, i64, i64, i64p, sp_type, C.POINTER(sp_type))
_sig("sp_type_hindexed_block", C.c_int, i64, i64, i64p, sp_type, C.POINTER(sp_type))
_sig("sp_type_struct", C.c_int, i64, i64p, i64p, C.POINTER(sp_type), C.POINTER(sp_type))
_sig("sp_type_resized", C.c_int, sp_type, i64, i64, C.POINTER(sp_type))
_sig("sp_type_lb", C.c_int, sp_type, i64p)
_sig("sp_type_free", C.c_int, sp_type)
_sig("sp_type_size", C.c_int, sp_type, i64p)
_sig("sp_type_extent", C.c_int, sp_type, i64p)
_sig("sp_type_commit", C.c_int, sp_type)
_sig("sp_type_query", C.c_int, sp_type, C.POINTER(TypeInfo), i64p, i64p, i64)
_sig("sp_type_flatten", C.c_int, sp_type, i64p, i64p, i64, i64p, C.POINTER(C.c_int))
_sig("sp_typefile_parse", C.c_int, C.c_char_p, C.POINTER(sp_type), C.c_char_p, i64)
_sig("sp_pack", C.c_int, C.c_void_p, u64, sp_type, i64, C.c_void_p, u64, i64p, C.c_void_p)
_sig("sp_unpack", C.c_int, C.c_void_p, u64, i64p, sp_type, i64, C.c_void_p, u64, C.c_void_p)
_sig("sp_pack_ex", C.c_int, C.c_void_p, u64, sp_type, i64, C.c_void_p, u64, i64p, C.c_void_p,
     C.POINTER(PackOptions))
_sig("sp_unpack_ex", C.c_int, C.c_void_p, u64, i64p, sp_type, i64, C.c_void_p, u64, C.c_void_p,
     C.POINTER(PackOptions))
_sig("sp_last_launch", C.c_int, C.POINTER(LaunchInfo))
_sig("sp_kernel_launch_count", i64)


def exported_symbols():
    """Every function include/stridepack_b200.h declares (for ABI tests)."""
    import re
    hdr = os.path.join(os.path.dirname(PKG_DIR), "include", "stridepack_b200.h")
    src = open(hdr).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sp_[a-z0-9_]+)\s*\(", src)))

# ---- model (perf_model.hpp / profile_io.hpp)
dbl = C.c_double
dblp = C.POINTER(C.c_double)
vp = C.c_void_p
_sig("sp_profile_create", C.c_int, C.POINTER(vp))
_sig("sp_profile_parse", C.c_int, C.c_char_p, C.POINTER(vp))
_sig("sp_profile_load", C.c_int, C.c_char_p, C.POINTER(vp))
_sig("sp_profile_save", C.c_int, vp, C.c_char_p, C.c_char_p, i64, i64p)
_sig("sp_profile_free", C.c_int, vp)
_sig("sp_profile_set_curve", C.c_int, vp, C.c_int, dblp, dblp, i64)
_sig("sp_profile_set_surface", C.c_int, vp, C.c_int, dblp, i64, dblp, i64, dblp)
_sig("sp_interp_1d", C.c_int, vp, C.c_int, dbl, dblp)
_sig("sp_interp_2d", C.c_int, vp, C.c_int, dbl, dbl, dblp)
_sig("sp_model_times", C.c_int, vp, i64, i64, dblp, dblp, dblp)
_sig("sp_choose_method", C.c_int, vp, i64, i64, C.POINTER(C.c_int))
_sig("sp_choose_method_b200", C.c_int, vp, i64, i64, C.c_int, C.POINTER(C.c_int), dblp)
_sig("sp_model_cache_create", C.c_int, vp, C.POINTER(vp))
_sig("sp_model_cache_choose", C.c_int, vp, i64, i64, C.POINTER(C.c_int))
_sig("sp_model_cache_free", C.c_int, vp)

# ---- batches
class BatchJob(C.Structure):
    _fields_ = [("src", C.c_void_p), ("src_bytes", u64), ("type", sp_type), ("count", i64),
                ("dst", C.c_void_p), ("dst_bytes", u64), ("position", i64)]


_sig("sp_batch_create", C.c_int, C.POINTER(BatchJob), i64, C.c_int, C.POINTER(vp))


class CopyJob(C.Structure):
    _fields_ = [("src", C.c_void_p), ("src_bytes", u64), ("src_type", sp_type), ("src_count", i64),
                ("dst", C.c_void_p), ("dst_bytes", u64), ("dst_type", sp_type), ("dst_count", i64)]


_sig("sp_copy_batch_create", C.c_int, C.POINTER(CopyJob), i64, C.POINTER(vp))
_sig("sp_copy", C.c_int, C.POINTER(CopyJob), vp)
_sig("sp_batch_execute", C.c_int, vp, vp)
_sig("sp_batch_bytes", C.c_int, vp, i64p)
_sig("sp_batch_free", C.c_int, vp)


# ---- halo
class HaloConfig(C.Structure):
    _fields_ = [("ranks", i64 * 3), ("interior", i64 * 3), ("radius", i64), ("element_bytes", i64)]


class HaloReport(C.Structure):
    _fields_ = [("pack_seconds", dbl), ("alltoallv_seconds", dbl), ("unpack_seconds", dbl),
                ("verified", i64), ("bytes_moved", i64), ("mismatched_cells", i64),
                ("measured_pack_seconds", dbl), ("measured_exchange_seconds", dbl),
                ("measured_unpack_seconds", dbl)]


_sig("sp_halo_types", C.c_int, C.POINTER(HaloConfig), C.POINTER(sp_type), C.POINTER(sp_type),
     C.POINTER(C.c_int), i64p)
_sig("sp_halo_neighbor", C.c_int, C.POINTER(HaloConfig), i64, C.POINTER(C.c_int), i64p)
_sig("sp_halo_fill", C.c_int, C.POINTER(HaloConfig), i64, vp, vp)
_sig("sp_halo_verify", C.c_int, C.POINTER(HaloConfig), i64, vp, vp, i64p)
_sig("sp_halo_run", C.c_int, C.POINTER(HaloConfig), vp, C.c_int, C.c_int, C.POINTER(HaloReport))

# ---- runtime
_sig("sp_rt_init", C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_int, i64, i64)
_sig("sp_rt_finalize", C.c_int)
_sig("sp_rt_rank", C.c_int, C.POINTER(C.c_int))
_sig("sp_rt_size", C.c_int, C.POINTER(C.c_int))
_sig("sp_rt_barrier", C.c_int)
_sig("sp_rt_host_send", C.c_int, C.c_int, C.c_int, vp, i64)
_sig("sp_rt_host_recv", C.c_int, C.c_int, C.c_int, vp, i64, i64p)
_sig("sp_rt_exchange_ptr", C.c_int, vp, C.POINTER(vp))
_sig("sp_rt_stream", C.c_int, C.POINTER(vp))
_sig("sp_rt_set_profile", C.c_int, vp)
_sig("sp_rt_choose", C.c_int, sp_type, i64, C.POINTER(C.c_int))
_sig("sp_rt_send", C.c_int, vp, u64, i64, sp_type, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int))
_sig("sp_rt_recv", C.c_int, vp, u64, i64, sp_type, C.c_int, C.c_int, i64p)
_sig("sp_rt_isend", C.c_int, vp, u64, i64, sp_type, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint64))
_sig("sp_rt_irecv", C.c_int, vp, u64, i64, sp_type, C.c_int, C.c_int, C.POINTER(C.c_uint64))
_sig("sp_rt_test", C.c_int, C.c_uint64, C.POINTER(C.c_int), i64p)
_sig("sp_rt_wait", C.c_int, C.c_uint64, i64p)
_sig("sp_rt_set_chunk", C.c_int, i64)
_sig("sp_rt_neighbor_alltoallv", C.c_int, vp, i64p, i64p, i64, C.POINTER(C.c_int), sp_type, vp, i64p, i64p, i64,
     C.POINTER(C.c_int), sp_type)
_sig("sp_rt_neighbor_alltoallw", C.c_int, vp, i64p, i64p, C.POINTER(sp_type), i64, C.POINTER(C.c_int), vp, i64p,
     i64p, C.POINTER(sp_type), i64, C.POINTER(C.c_int))
_sig("sp_rt_neighbor_alltoallw_init", C.c_int, vp, i64p, i64p, C.POINTER(sp_type), i64, C.POINTER(C.c_int), vp,
     i64p, i64p, C.POINTER(sp_type), i64, C.POINTER(C.c_int), C.POINTER(vp))
_sig("sp_nbr_plan_start", C.c_int, vp)
_sig("sp_nbr_plan_test", C.c_int, vp, C.POINTER(C.c_int))
_sig("sp_nbr_plan_wait", C.c_int, vp)
_sig("sp_nbr_plan_free", C.c_int, vp)
_sig("sp_halo_plan_create", C.c_int, C.POINTER(HaloConfig), vp, C.c_int, C.POINTER(vp))
_sig("sp_halo_plan_exchange", C.c_int, vp, dblp)
_sig("sp_halo_plan_free", C.c_int, vp)
