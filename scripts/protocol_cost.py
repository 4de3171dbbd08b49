"""What the in-kernel completion protocol costs, measured on ONE GPU.

At one rank the halo plan drops its self edges (no flags). With
SPB_HALO_SELF_FLAGS set the self edges keep the full protocol (FREE pre-store
and wait, READY signal, block-0 post wait), so the difference between the two
plans is the protocol's cost at the kernel tail. Run it against two builds
(SPB_LIB=...) to compare epilogue designs. Cold L2 before each timed
exchange, as in the bench; one JSON line per (method, flags).
"""
import json
import os
import statistics
import sys
import uuid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2012_14363_b200.halo as H  # noqa: E402
import paper_2012_14363_b200.rt as rt  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 30
tag = os.environ.get("PROTO_TAG", os.path.basename(os.environ.get("SPB_LIB", "current")))
rt.init(0, 1, "pc" + uuid.uuid4().hex[:8], device=0, window_bytes=1 << 20, host_bytes=1 << 20)
cfg = H.HaloConfig((1, 1, 1), (256, 256, 256), 2, 32)
alloc = torch.empty(260 ** 3 * 32, dtype=torch.uint8, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
sink = torch.empty(1, dtype=torch.int64, device="cuda")
rs = torch.cuda.ExternalStream(rt.stream())


def cold(i):
    with torch.cuda.stream(rs):
        flush.fill_(i & 0xFF)
        torch.sum(flush.view(torch.int64), dim=0, out=sink[0])


for method, name in ((H.DIRECT, "direct"), (H.FUSED_ASYNC, "fused_async")):
    for flags in (False, True):
        if flags:
            os.environ["SPB_HALO_SELF_FLAGS"] = "1"
        else:
            os.environ.pop("SPB_HALO_SELF_FLAGS", None)
        H.fill(cfg, 0, alloc)
        torch.cuda.synchronize()
        plan = rt.HaloPlan(cfg, alloc, method)
        for i in range(5):
            cold(i)
            plan.exchange()
        ts = []
        for i in range(iters):
            cold(i)
            ts.append(plan.exchange()["iteration"] * 1e6)
        # back to back, enqueue only (no flush): the pipelined rate
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(rs)
        for i in range(iters):
            plan.exchange(timed=False)
        b.record(rs)
        torch.cuda.synchronize()
        bad = H.verify(cfg, 0, alloc)
        plan.free()
        print(json.dumps({"build": tag, "method": name, "self_flags": flags,
                          "cold_us_median": round(statistics.median(ts), 2), "cold_us_min": round(min(ts), 2),
                          "back_to_back_us": round(a.elapsed_time(b) * 1e3 / iters, 2), "bad": int(bad)}))
rt.finalize()
