"""Model + halo golden fixtures from the reference (called by make_golden.py).

  default.profile    proj/data/default.profile after the reference's
                     load_profile -> save_profile round trip
  model_golden.json  reference choose_method + three model times on the
                     acceptance grid (acceptance.cpp:217-230), random queries
                     and two scaled profiles (test_util.hpp:153-167)
  halo_golden.json   reference halo region programs (halo.hpp:98-130) and
                     run_exchange reports (halo.hpp:172-322)
"""
import ctypes as C
import json
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PROFILE = "/root/reference/proj/data/default.profile"


def _save(R, h, header=""):
    need = R.lib.ref_profile_save(h, header.encode(), None, 0)
    buf = C.create_string_buffer(-need)
    n = R.lib.ref_profile_save(h, header.encode(), buf, -need)
    assert n >= 0
    return buf.value.decode()


def _choose(R, h, o, b):
    m = C.c_int()
    td, to, ts = C.c_double(), C.c_double(), C.c_double()
    st = R.lib.ref_choose(h, o, b, C.byref(m), C.byref(td), C.byref(to), C.byref(ts))
    if st:
        return {"o": o, "b": b, "status": st}
    return {"o": o, "b": b, "status": 0, "method": m.value, "t_device": td.value,
            "t_oneshot": to.value, "t_staged": ts.value}


def acceptance_grid():
    grid = []
    for i in range(20):
        for j in range(20):
            obj = 256.0 * math.pow(64.0 * 1024 * 1024 / 256.0, i / 19.0)
            blk = 8.0 * math.pow(4096.0 / 8.0, j / 19.0)
            o = int(obj)
            grid.append((o, min(int(blk), o)))
    return grid


def main(R):
    st = C.c_int()
    h = R.lib.ref_profile_load(REF_PROFILE.encode(), C.byref(st))
    assert st.value == 0
    text = _save(R, h, "proj/data/default.profile as re-emitted by the reference's save_profile\n"
                       "(synthetic Summit-shaped fixture, see the reference header)")
    with open(os.path.join(HERE, "default.profile"), "w") as f:
        f.write(text)
    rng = np.random.default_rng(8)
    queries = acceptance_grid()
    queries += [(int(o), int(1 + rng.integers(0, o))) for o in rng.integers(1, 4 << 20, 300)]
    queries += [(64 << k, min(8 << j, 64 << k)) for k in range(20) for j in range(10)]
    queries += [(0, 1), (64, 0), (64, 128)]  # validation errors
    out = {"base": [_choose(R, h, o, b) for o, b in queries], "scaled": {}}
    for k in (0.5, 3.0):
        hs = R.lib.ref_profile_scaled(h, k)
        out["scaled"][str(k)] = [_choose(R, hs, o, b) for o, b in queries[:400]]
        R.lib.ref_profile_free(hs)
    with open(os.path.join(HERE, "model_golden.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))

    # halo
    halo = {"types": [], "reports": []}
    for interior, radius, elem in [((16, 16, 16), 3, 64), ((256, 256, 256), 2, 32), ((4, 6, 8), 2, 4),
                                   ((2, 2, 2), 1, 8), ((8, 8, 8), 2, 16)]:
        arr = (C.c_int64 * 3)(*interior)
        need = R.lib.ref_halo_types(arr, radius, elem, None, 0)
        buf = np.zeros(-need, np.int64)
        got = R.lib.ref_halo_types(arr, radius, elem, buf.ctypes.data_as(C.POINTER(C.c_int64)), len(buf))
        assert got == -need
        regions, at = [], 0
        while at < got:
            d = buf[at:at + 3].tolist()
            cells = int(buf[at + 3])
            at += 4
            ln = int(buf[at])
            send = buf[at + 1:at + 1 + ln].tolist()
            at += 1 + ln
            ln = int(buf[at])
            recv = buf[at + 1:at + 1 + ln].tolist()
            at += 1 + ln
            regions.append({"dir": d, "cells": cells, "send": send, "recv": recv})
        halo["types"].append({"interior": interior, "radius": radius, "elem": elem, "regions": regions})

    class Rep(C.Structure):
        _fields_ = [("pack", C.c_double), ("xfer", C.c_double), ("unpack", C.c_double),
                    ("verified", C.c_int64), ("bytes", C.c_int64)]

    for ranks, interior, radius, elem in [((1, 1, 1), (16, 16, 16), 3, 64), ((2, 2, 2), (16, 16, 16), 3, 64),
                                          ((2, 2, 2), (8, 8, 8), 2, 16), ((3, 1, 2), (4, 6, 8), 2, 4),
                                          ((1, 1, 1), (6, 6, 6), 1, 8), ((2, 1, 1), (6, 6, 6), 1, 8),
                                          ((2, 1, 1), (6, 6, 6), 1, 16), ((3, 3, 3), (16, 16, 16), 3, 64)]:
        rep = Rep()
        st = R.lib.ref_run_exchange((C.c_int64 * 3)(*ranks), (C.c_int64 * 3)(*interior), radius, elem, h,
                                    C.byref(rep))
        assert st == 0
        halo["reports"].append({"ranks": ranks, "interior": interior, "radius": radius, "elem": elem,
                                "pack": rep.pack, "alltoallv": rep.xfer, "unpack": rep.unpack,
                                "verified": rep.verified, "bytes": rep.bytes})
    with open(os.path.join(HERE, "halo_golden.json"), "w") as f:
        json.dump(halo, f, separators=(",", ":"))
    R.lib.ref_profile_free(h)
    print(f"model: {len(out['base'])} queries; halo: {len(halo['types'])} geometries, "
          f"{len(halo['reports'])} reports")
