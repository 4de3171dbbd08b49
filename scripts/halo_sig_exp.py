"""Timing study of the DIRECT halo plan's in-kernel protocol on one rank:
SPB_HALO_EXPERIMENT bits drop the block wait (1), the pre-signal (2), the
last block's post-wait (4), the release signal (8). One rank only."""
import os, sys, json, uuid, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2012_14363_b200.halo as H
import paper_2012_14363_b200.rt as rt
torch.cuda.set_device(0)
rt.init(0, 1, uuid.uuid4().hex[:8], device=0, window_bytes=1 << 20, host_bytes=1 << 20)
cfg = H.HaloConfig((1, 1, 1), (256, 256, 256), 2, 32)
alloc = torch.empty(260 ** 3 * 32, dtype=torch.uint8, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
sink = torch.empty(1, dtype=torch.int64, device="cuda")
st = torch.cuda.ExternalStream(rt.stream())
out = {}
for bits in [0, 1, 2, 4, 12, 15]:
    os.environ["SPB_HALO_EXPERIMENT"] = str(bits)
    H.fill(cfg, 0, alloc)
    torch.cuda.synchronize()
    plan = rt.HaloPlan(cfg, alloc, H.DIRECT)
    ts = []
    for i in range(25):
        with torch.cuda.stream(st):
            flush.fill_(i & 0xFF)
            torch.sum(flush.view(torch.int64), dim=0, out=sink[0])
        t = plan.exchange()
        if i >= 5:
            ts.append(t["iteration"] * 1e6)
    plan.free()
    out[bits] = round(statistics.median(ts), 2)
print(json.dumps(out))
rt.finalize()
