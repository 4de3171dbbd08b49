"""Multi-rank runs on ONE B200 under MPS (scripts/gpu_r02l.sh starts the
daemon): N processes share cuda:0 and their kernels run concurrently, so the
completion protocol between ranks (FREE/READY flags written across
processes through CUDA IPC, block-0 post waits, the neighbour-call entry
protocol) runs with real concurrency instead of time slicing. The data path
is local HBM, not NVLink: the numbers show the protocol and the shared-HBM
behaviour, not link bandwidth. Launched by torchrun with gloo.

Per method, steady state: every rank enqueues ITERS exchanges back to back
(enqueue only, device-ordered), timed with events on its runtime stream,
max over ranks. The N ranks together move N x 25.6 MB each way per
iteration through the one GPU's HBM, so `aggregate_hbm_GBps` (read + write
bytes of all ranks / iteration time) is the number to compare with the
single-rank iteration. The MPI_Neighbor_alltoallw form is host-synchronous:
its per-call wall time is the mean over ITERS calls. At N=2 the send
section of bench.py runs too.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2012_14363_b200.halo as H  # noqa: E402
import paper_2012_14363_b200.rt as rt  # noqa: E402
from bench_parts import GRIDS, send_section  # noqa: E402

ITERS = int(os.environ.get("MPS_ITERS", "50"))
rank = int(os.environ["RANK"])
world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
name = ["mps" + os.urandom(5).hex()]
dist.broadcast_object_list(name, src=0)


def vmax(v):
    t = torch.tensor([float(v)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


grid = GRIDS[world]
cfg = H.HaloConfig(grid, (256, 256, 256), 2, 32)
regions = H.build_halo_types(cfg)
seg = sum(r.send.size for r in regions)
rt.init(rank, world, name[0], device=0, window_bytes=1 << 20, host_bytes=1 << 20)
alloc = torch.empty(260 ** 3 * 32, dtype=torch.uint8, device="cuda")
rs = torch.cuda.ExternalStream(rt.stream())
out = {"world": world, "grid": list(grid), "device": "cuda:0 shared by every rank (MPS)",
       "mps": os.environ.get("CUDA_MPS_PIPE_DIRECTORY") is not None,
       "flag_waits": os.environ.get("TEMPI_FLAG_WAIT", "auto (stream: ranks share a GPU)"),
       "bytes_per_rank": seg, "iters": ITERS}
for mname, method in (("direct", H.DIRECT), ("fused_async", H.FUSED_ASYNC)):
    H.fill(cfg, rank, alloc)
    torch.cuda.synchronize()
    rt.barrier()
    plan = rt.HaloPlan(cfg, alloc, method)
    for _ in range(5):
        plan.exchange(timed=False)
    rs.synchronize()
    rt.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(rs)
    for _ in range(ITERS):
        plan.exchange(timed=False)
    b.record(rs)
    rs.synchronize()
    it_us = vmax(a.elapsed_time(b) * 1e3 / ITERS)
    bad = vmax(H.verify(cfg, rank, alloc))
    plan.free()
    traffic = (2 if mname == "direct" else 4) * seg * world  # HBM bytes of all ranks per iteration
    out[mname] = {"iteration_us": round(it_us, 2), "verified": bad == 0,
                  "aggregate_hbm_GBps": round(traffic / (it_us * 1e-6) / 1e9, 1)}
# MPI_Neighbor_alltoallw with the 26 region types (host-synchronous calls)
H.fill(cfg, rank, alloc)
torch.cuda.synchronize()
sends = [(H.neighbor(cfg, rank, r.dir), 1, r.send, 0) for r in regions]
recvs = [(H.neighbor(cfg, rank, tuple(-x for x in r.dir)), 1, regions[25 - j].recv, 0)
         for j, r in enumerate(regions)]
nw = rt.NeighborW(sends, recvs)
for _ in range(5):
    nw(alloc, alloc)
rt.barrier()
t0 = time.perf_counter()
for _ in range(ITERS):
    nw(alloc, alloc)
call_us = vmax((time.perf_counter() - t0) / ITERS * 1e6)
out["alltoallw"] = {"call_us": round(call_us, 2), "verified": vmax(H.verify(cfg, rank, alloc)) == 0,
                    "aggregate_hbm_GBps": round(2 * seg * world / (call_us * 1e-6) / 1e9, 1)}
rt.finalize()
if world == 2 and os.environ.get("MPS_SEND", "1") == "1":
    out["send"] = send_section(torch, rank, world, 0, name[0])
dist.barrier()
if rank == 0:
    print(json.dumps(out), flush=True)
dist.destroy_process_group()
