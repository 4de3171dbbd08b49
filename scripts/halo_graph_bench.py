"""Halo exchange (config 5: 256^3, r = 2, 32 B, one rank) enqueued eagerly
vs replayed from a CUDA graph: wall time per iteration of 200 iterations
(200 eager enqueues, or 20 replays of a graph holding 10 exchanges), each
run synchronised once at the end. DIRECT and FUSED_ASYNC. One JSON line per
method.

  python scripts/halo_graph_bench.py
"""
import json
import os
import sys
import time
import uuid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2012_14363_b200.halo as H  # noqa: E402
import paper_2012_14363_b200.rt as rt  # noqa: E402


def main():
    torch.cuda.set_device(0)
    rt.init(0, 1, "hg" + uuid.uuid4().hex[:8], device=0, window_bytes=1 << 20, host_bytes=1 << 20)
    cfg = H.HaloConfig((1, 1, 1), (256, 256, 256), 2, 32)
    alloc = torch.empty(260 ** 3 * 32, dtype=torch.uint8, device="cuda")
    rs = torch.cuda.ExternalStream(rt.stream())
    for method, name in ((H.DIRECT, "direct"), (H.FUSED_ASYNC, "fused_async")):
        H.fill(cfg, 0, alloc)
        torch.cuda.synchronize()
        plan = rt.HaloPlan(cfg, alloc, method)
        for _ in range(5):
            plan.exchange(timed=False)
        rs.synchronize()
        t0 = time.perf_counter()
        for _ in range(200):
            plan.exchange(timed=False)
        enq = time.perf_counter() - t0
        rs.synchronize()
        eager = time.perf_counter() - t0
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(rs):
            g.capture_begin()
            for _ in range(10):
                plan.exchange(timed=False)
            g.capture_end()
            g.replay()
        rs.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(rs):
            for _ in range(20):
                g.replay()
        genq = time.perf_counter() - t0
        rs.synchronize()
        graph = time.perf_counter() - t0
        H.fill(cfg, 0, alloc)
        torch.cuda.synchronize()
        with torch.cuda.stream(rs):
            g.replay()
        rs.synchronize()
        bad = H.verify(cfg, 0, alloc)
        print(json.dumps({"method": name, "iterations": 200,
                          "eager_us_per_iteration": round(eager / 200 * 1e6, 2),
                          "eager_host_enqueue_us_per_iteration": round(enq / 200 * 1e6, 2),
                          "graph_us_per_iteration": round(graph / 200 * 1e6, 2),
                          "graph_host_enqueue_us_per_iteration": round(genq / 200 * 1e6, 2),
                          "verified_after_replay": bad == 0}), flush=True)
        del g
        plan.free()
    rt.finalize()


if __name__ == "__main__":
    main()
