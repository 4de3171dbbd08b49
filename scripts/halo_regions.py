"""Halo (BASELINE config 5, one rank) kernel study, cold clean L2 before
every timed launch: each region class packed alone through sp_pack (k_words),
the 26-region pack batch, the 26-region DIRECT copy batch, and a plain
device copy of the same byte count for calibration."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2012_14363_b200 as sp
import paper_2012_14363_b200.halo as H

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = H.HaloConfig((1, 1, 1), (256, 256, 256), 2, 32)
regs = H.build_halo_types(cfg)
pad = 260 ** 3 * 32
alloc = torch.empty(pad, dtype=torch.uint8, device="cuda")
H.fill(cfg, 0, alloc)
seg = [0]
for r in regs:
    seg.append(seg[-1] + r.send.size)
buf = torch.empty(seg[-1], dtype=torch.uint8, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
sink = torch.empty(1, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()


def timed(fn):
    ts = []
    for i in range(reps):
        flush.fill_(i & 0xFF)
        torch.sum(flush.view(torch.int64), dim=0, out=sink[0])  # same stream, not waited for:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)  # no host latency timed
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return min(ts)


out = {}
for name, pick in (("x-face", lambda r: r.dir == (1, 0, 0)), ("y-face", lambda r: r.dir == (0, 1, 0)),
                   ("z-face", lambda r: r.dir == (0, 0, 1))):
    r = [r for r in regs if pick(r)][0]
    us = timed(lambda: sp.pack(alloc, r.send, 1, buf, 0))
    out[name] = {"bytes": r.send.size, "us": round(us, 2), "GBps": round(2 * r.send.size / us / 1e3, 1),
                 "kernel": sp.last_launch().kernel.name}
pb = H.Batch([(alloc, r.send, 1, buf, seg[j]) for j, r in enumerate(regs)])
us = timed(pb.execute)
out["pack26"] = {"bytes": seg[-1], "us": round(us, 2), "GBps": round(2 * seg[-1] / us / 1e3, 1)}
ub = H.Batch([(buf, r.recv, 1, alloc, seg[j]) for j, r in enumerate(regs)], unpack=True)
us = timed(ub.execute)
out["unpack26"] = {"bytes": seg[-1], "us": round(us, 2), "GBps": round(2 * seg[-1] / us / 1e3, 1)}
cb = H.Batch.copies([(alloc, r.send, 1, alloc, regs[25 - j].recv, 1) for j, r in enumerate(regs)])
us = timed(cb.execute)
out["direct26"] = {"bytes": seg[-1], "us": round(us, 2), "GBps": round(2 * seg[-1] / us / 1e3, 1)}
dst = torch.empty_like(buf)
src = alloc[: seg[-1]]
us = timed(lambda: dst.copy_(src))
out["memcpy"] = {"bytes": seg[-1], "us": round(us, 2), "GBps": round(2 * seg[-1] / us / 1e3, 1)}
print(json.dumps(out, indent=1))
