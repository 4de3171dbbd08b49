import os, sys, statistics, uuid
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2012_14363_b200.halo as H
import paper_2012_14363_b200.rt as rt
rt.init(0, 1, "exp" + uuid.uuid4().hex[:8], device=0, window_bytes=1 << 20, host_bytes=1 << 20)
cfg = H.HaloConfig((1, 1, 1), (256, 256, 256), 2, 32)
alloc = torch.empty(260 ** 3 * 32, dtype=torch.uint8, device="cuda")
H.fill(cfg, 0, alloc)
for method in (H.FUSED, H.FUSED_ASYNC):
    plan = rt.HaloPlan(cfg, alloc, method)
    for _ in range(5):
        plan.exchange()
    ts = [plan.exchange() for _ in range(20)]
    print(method, os.environ.get("SPB_EXP_NOWAIT"), os.environ.get("SPB_EXP_NOSIGNAL"),
          {k: round(statistics.median(t[k] for t in ts) * 1e6, 2) for k in ts[0]}, "bad", H.verify(cfg, 0, alloc))
    plan.free()
rt.finalize()
