"""Profiling driver: runs pack/unpack of the cfg2 object for chosen E0s with
incount K, L2 flushed before each kernel; prints per-kernel event timings and
a same-size plain device copy for calibration. Used under ncu and alone.

  python scripts/prof_cfg2.py --e0 512,32,8,1 --k 32 --reps 3 [--unpack]
"""
import argparse
import ctypes as C
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2012_14363_b200 as sp  # noqa: E402
from paper_2012_14363_b200 import _capi  # noqa: E402


def prog(e0):
    e2 = 2 ** math.ceil(math.log2((1 << 20) // e0) / 2)
    e1 = (1 << 20) // (e0 * e2)
    return [4, 3, 0, 1024, 1024, 1024, e0, e1, e2, 0, 0, 0, 0, 0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--e0", default="512,32,8,1")
    ap.add_argument("--k", type=int, default=32)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--mode", default="both", choices=["pack", "unpack", "both"])
    ap.add_argument("--kernel", type=int, default=0)
    ap.add_argument("--copy", action="store_true")
    a = ap.parse_args()
    K = a.k
    lib = _capi.lib
    s = torch.cuda.current_stream()
    sh = C.c_void_p(s.cuda_stream)
    src = torch.empty(K << 30, dtype=torch.uint8, device="cuda")
    src[::4099] = 1
    packed = torch.zeros(K << 20, dtype=torch.uint8, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    opt = _capi.PackOptions(1, a.kernel, 0)
    pos = C.c_int64(0)
    for e0 in [int(x) for x in a.e0.split(",")]:
        ct = sp.commit_type(sp.from_program(prog(e0)))
        for pk in (True, False):
            if (a.mode == "pack" and not pk) or (a.mode == "unpack" and pk):
                continue
            ts = []
            for _ in range(a.reps):
                flush.fill_(1)
                torch.sum(flush.view(torch.int64))
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ev0.record(s)
                pos.value = 0
                if pk:
                    st = lib.sp_pack_ex(src.data_ptr(), src.numel(), ct.handle, K, packed.data_ptr(),
                                        packed.numel(), C.byref(pos), sh, C.byref(opt))
                else:
                    st = lib.sp_unpack_ex(packed.data_ptr(), packed.numel(), C.byref(pos), ct.handle, K,
                                          src.data_ptr(), src.numel(), sh, C.byref(opt))
                assert st == 0, lib.sp_last_error()
                ev1.record(s)
                torch.cuda.synchronize()
                ts.append(ev0.elapsed_time(ev1))
            li = sp.last_launch()
            us = min(ts) * 1e3
            print(f"E0={e0:4d} {'pack  ' if pk else 'unpack'} K={K} {li.kernel.name}/w{li.word} grid={li.grid} "
                  f"min {us:8.2f} us  {2 * K * (1 << 20) / (us * 1e-6) / 1e9:8.1f} GB/s", flush=True)
    if a.copy:
        dst2 = torch.empty(K << 20, dtype=torch.uint8, device="cuda")
        srcc = src[: K << 20]
        for _ in range(a.reps):
            flush.zero_()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(s)
            dst2.copy_(srcc)
            ev1.record(s)
            torch.cuda.synchronize()
            us = ev0.elapsed_time(ev1) * 1e3
        print(f"plain copy {K} MiB: {us:.2f} us {2 * K * (1 << 20) / (us * 1e-6) / 1e9:.1f} GB/s")


if __name__ == "__main__":
    main()
