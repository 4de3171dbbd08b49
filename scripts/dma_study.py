"""Copy engines vs SM kernels for pack/unpack (future work:
"evaluate the use of the GPU DMA engine for non-contiguous data (e.g.
cudaMemcpy2D)"). For the cfg2 object at each E0, K objects per call, L2
flushed before every call, CUDA events on the launching stream, best of
--reps:
  * device -> device: the automatic kernel choice vs Kernel.DMA
    (cudaMemcpy3DAsync, no SM involved);
  * device -> pinned host (pack) and pinned host -> device (unpack): the
    engine's default (kernel into a device stage + chunked DMA of the
    packed bytes) vs Kernel.DMA straight between the strided device layout
    and host memory.
One JSON line per (E0, case).

  python scripts/dma_study.py --e0 1,8,32,64,128,512 --k 16 --reps 3
"""
import argparse
import ctypes as C
import json
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
    ap.add_argument("--e0", default="1,2,4,8,16,32,64,128,256,512")
    ap.add_argument("--k", type=int, default=16)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    K = a.k
    lib = _capi.lib
    s = torch.cuda.current_stream()
    sh = C.c_void_p(s.cuda_stream)
    strided = torch.empty(K << 30, dtype=torch.uint8, device="cuda")
    strided[::4099] = 1
    packed = torch.zeros(K << 20, dtype=torch.uint8, device="cuda")
    pinned = torch.zeros(K << 20, dtype=torch.uint8).pin_memory()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    pos = C.c_int64(0)

    def timed(fn):
        best = None
        for _ in range(a.reps):
            flush.fill_(1)
            torch.sum(flush.view(torch.int64))
            e0_, e1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0_.record(s)
            fn()
            e1_.record(s)
            e1_.synchronize()
            t = e0_.elapsed_time(e1_) * 1e3
            best = t if best is None else min(best, t)
        return best

    for e0 in [int(x) for x in a.e0.split(",")]:
        ct = sp.commit_type(sp.from_program(prog(e0)))
        nbytes = K * ct.size
        for case, pk, buf in (("d2d pack", True, packed), ("d2d unpack", False, packed),
                              ("pack to pinned", True, pinned), ("unpack from pinned", False, pinned)):
            row = {"E0": e0, "K": K, "case": case, "bytes": nbytes}
            for name, kernel in (("kernels", 0), ("dma", sp.Kernel.DMA)):
                opt = _capi.PackOptions(1, int(kernel), 0)

                def call():
                    pos.value = 0
                    if pk:
                        st = lib.sp_pack_ex(strided.data_ptr(), strided.numel(), ct.handle, K, buf.data_ptr(),
                                            buf.numel(), C.byref(pos), sh, C.byref(opt))
                    else:
                        st = lib.sp_unpack_ex(buf.data_ptr(), buf.numel(), C.byref(pos), ct.handle, K,
                                              strided.data_ptr(), strided.numel(), sh, C.byref(opt))
                    if st:
                        raise RuntimeError(f"status {st}: {lib.sp_last_error().decode()}")

                try:
                    us = timed(call)
                    row[name + "_us"] = round(us, 2)
                    # HBM-side algorithmic bytes: read + write of the described bytes
                    row[name + "_GBps"] = round(2 * nbytes / us / 1e3, 1)
                except RuntimeError as exc:
                    row[name + "_error"] = str(exc)[:120]
            if "kernels_us" in row and "dma_us" in row:
                row["dma_over_kernels"] = round(row["dma_us"] / row["kernels_us"], 2)
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
