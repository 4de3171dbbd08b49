"""Typed-copy kernels against pack/unpack on the same 64 MiB objects (cold
clean L2 before every launch, events on the launching stream, min of 7):
  pack    sp_pack (k_words / k_smallrow)     strided -> packed
  unpack  sp_unpack                          packed  -> strided
  copy    sp_copy (k_job, one job by value)  strided -> strided (same type)
  batch   Batch.copies (k_batchp, 1 job)     strided -> strided
GB/s counts read + write of the described bytes."""
import json, math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2012_14363_b200 as sp
from paper_2012_14363_b200.halo import Batch

def cfg4(e0, n):
    rows = n // e0
    e2 = 2 ** (int(math.log2(rows)) // 2)
    e1 = rows // e2
    return [4, 3, 0, max(2 * e0, 64), 2 * e1, e2, e0, e1, e2, 0, 0, 0, 0, 0]

s = torch.cuda.current_stream()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
sink = torch.empty(1, dtype=torch.int64, device="cuda")

def timed(fn, reps=7):
    ts = []
    for i in range(reps):
        flush.fill_(i & 0xFF)
        torch.sum(flush.view(torch.int64), dim=0, out=sink[0])
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); fn(); b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return min(ts)

out = {}
for e0 in (8, 64, 512):
    ct = sp.commit_type(sp.from_program(cfg4(e0, 64 << 20)))
    src = torch.empty(ct.span, dtype=torch.uint8, device="cuda")
    dst = torch.empty(ct.span, dtype=torch.uint8, device="cuda")
    pk = torch.empty(ct.size, dtype=torch.uint8, device="cuda")
    b = Batch.copies([(src, ct, 1, dst, ct, 1)])
    r = {}
    for name, fn in (("pack", lambda: sp.pack(src, ct, 1, pk, 0)), ("unpack", lambda: sp.unpack(pk, 0, ct, 1, dst)),
                     ("copy", lambda: sp.copy(src, ct, 1, dst, ct, 1)), ("batch", b.execute)):
        us = timed(fn)
        r[name] = {"us": round(us, 2), "GBps": round(2 * ct.size / us / 1e3, 1)}
    out[f"E0={e0}"] = r
print(json.dumps(out, indent=1))
