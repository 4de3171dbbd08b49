"""Misaligned long rows: the funnel-shift kernel against the word kernel the
alignment would otherwise force (W = 1/2/4), and against the same shape with
aligned rows as the ceiling. Rows of c0 bytes at pitch 2*c0 + pad; ~256 MiB
packed per launch, L2 flushed before each launch, CUDA-event timing.

  python scripts/shift_bench.py [--c0 16,32,64,100,128,256,1024] [--reps 5]
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2012_14363_b200 as sp  # noqa: E402
from paper_2012_14363_b200 import _capi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c0", default="16,32,64,100,128,256,1024")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--packed-mib", type=int, default=256)
    a = ap.parse_args()
    lib = _capi.lib
    s = torch.cuda.current_stream()
    sh = C.c_void_p(s.cuda_stream)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    nbytes = a.packed_mib << 20
    packed = torch.zeros(nbytes + 64, dtype=torch.uint8, device="cuda")
    src = torch.empty(2 * nbytes + (64 << 20), dtype=torch.uint8, device="cuda")
    src[::4099] = 3
    pos = C.c_int64(0)
    out = []
    for c0 in [int(x) for x in a.c0.split(",")]:
        rows = nbytes // c0
        for pad, shift in ((0, 0), (1, 0), (0, 1), (4, 4)):
            pitch = 2 * c0 + pad
            ct = sp.commit_type(sp.from_program([3, rows, 1, pitch, 1, c0, 0, 0]))
            sb = src[shift:]
            for kernel in (1, 7):
                for pk in (True, False):
                    ts = []
                    li = None
                    for _ in range(a.reps):
                        flush.fill_(1)
                        torch.sum(flush.view(torch.int64))
                        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        opt = _capi.PackOptions(1, kernel, 0)
                        ev0.record(s)
                        pos.value = 0
                        if pk:
                            st = lib.sp_pack_ex(sb.data_ptr(), sb.numel(), ct.handle, 1, packed.data_ptr(),
                                                packed.numel(), C.byref(pos), sh, C.byref(opt))
                        else:
                            st = lib.sp_unpack_ex(packed.data_ptr(), packed.numel(), C.byref(pos), ct.handle, 1,
                                                  sb.data_ptr(), sb.numel(), sh, C.byref(opt))
                        ev1.record(s)
                        if st != 0:
                            raise RuntimeError(f"status {st} c0={c0} kernel={kernel}")
                        torch.cuda.synchronize()
                        ts.append(ev0.elapsed_time(ev1))
                        li = sp.last_launch()
                    ms = sorted(ts)[len(ts) // 2]
                    rec = dict(c0=c0, pitch=pitch, shift=shift, kernel=int(li.kernel), word=li.word,
                               dir="pack" if pk else "unpack", ms=round(ms, 4),
                               gbps=round(2 * rows * c0 / ms / 1e6, 1))
                    print(json.dumps(rec), flush=True)
                    out.append(rec)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "shift_bench.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
