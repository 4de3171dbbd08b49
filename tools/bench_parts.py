"""Multi-GPU sections of bench.py (imported by it; also runnable alone).

halo_section : the 3D 26-neighbour halo exchange (BASELINE config 5: radius
               2, 256^3 points/rank, 32 B/point) on a rank grid of the
               world size, through the engine's fused pack-to-peer plan
               (one batch launch per rank stores every segment into the
               neighbour's HBM over CUDA IPC / NVLink), verified cell by
               cell, and -- when torch.distributed is up -- the NCCL
               baseline (batch pack, 26 ncclSend/ncclRecv in one group,
               batch unpack). Device-timed with CUDA events, max over ranks.
send_section : BASELINE config 4, a non-contiguous 3D object sent rank 0 ->
               rank 1 (half ping-pong), 1 KiB-64 MiB, every
               fixed method and the model's choice.
"""
from __future__ import annotations

import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GRIDS = {1: (1, 1, 1), 2: (2, 1, 1), 4: (2, 2, 1), 8: (2, 2, 2), 3: (3, 1, 1), 6: (3, 2, 1)}
NVLINK_GBPS = 900.0          # per direction per GPU, nominal
NVLINK_FALLBACK_GBPS = 770.0  # B200_PROFILING.md's peer-copy figure: used only when no peer GPU is visible


def nvlink_peak(torch, local, peer, nbytes=256 << 20, reps=10):
    """one-way NVLink bandwidth measured in this run: cudaMemcpyPeerAsync
    (torch's cross-device copy) of `nbytes` from device `local` to device
    `peer`, CUDA events on the copying stream, best of `reps`. Also enables
    peer access between the two devices for this process."""
    src = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{local}")
    dst = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{peer}")
    s = torch.cuda.current_stream(local)
    best = None
    for i in range(reps + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        dst.copy_(src, non_blocking=True)
        b.record(s)
        b.synchronize()
        if i >= 2:
            t = a.elapsed_time(b) * 1e-3
            best = t if best is None else min(best, t)
    del src, dst
    return nbytes / best / 1e9


def calibrate_peer(torch, prof, local, peer, reps=5):
    """Measure, on THIS box, the two model terms that involve a peer GPU and
    put them into `prof` (a MachineProfile): the gpu_gpu curve (a plain
    cudaMemcpyPeerAsync of n bytes) and the gpu_direct_peer surface (one
    typed copy of the profile probe hvector(o/b,1,2b,contiguous(b)) from this
    GPU into the same layout on the peer, the DIRECT method). Same grids and
    timing rule as tools/measure_profile: median wall time of synchronous
    calls."""
    import time
    import paper_2012_14363_b200 as sp
    objects = [1 << k for k in range(10, 27, 2)]
    blocks = [1, 4, 16, 64, 256, 1024, 4096]
    big = objects[-1]
    src = torch.zeros(2 * big, dtype=torch.uint8, device=f"cuda:{local}")
    dst = torch.zeros(2 * big, dtype=torch.uint8, device=f"cuda:{peer}")
    B = sp.make_named(sp.NamedKind.Byte)
    s = torch.cuda.current_stream(local)

    def med(fn):
        for _ in range(2):
            fn()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts)

    grid = []
    for o in objects:
        row = []
        for b0 in blocks:
            b = min(b0, o)
            ct = sp.commit_type(sp.make_hvector(o // b, 1, 2 * b, sp.make_contiguous(b, B)))
            row.append(med(lambda: sp.copy(src, ct, 1, dst, ct, 1, stream=s, sync=True)))
        grid.append(row)
    prof.set_surface("gpu_direct_peer", objects, blocks, grid)
    sizes = [64 << k for k in range(21)]
    curve = []
    for n in sizes:
        def cp():
            dst[:n].copy_(src[:n], non_blocking=True)
            s.synchronize()
        curve.append(med(cp))
    prof.set_curve("gpu_gpu", sizes, curve)
    del src, dst
    torch.cuda.empty_cache()
    return {"gpu_direct_peer_1MiB_64B_us": round(grid[objects.index(1 << 20)][blocks.index(64)] * 1e6, 2),
            "gpu_gpu_64MiB_us": round(curve[-1] * 1e6, 1)}


def _hbm_peak():
    """measured HBM copy bandwidth (MEASURED_PEAKS.json), else the recipe's fallback"""
    import json
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f).get("hbm_gbs", 6650.0))
    return 6650.0


def remote_bytes(cfg, regions, rank):
    """bytes this rank sends to OTHER ranks (NVLink traffic)"""
    import paper_2012_14363_b200.halo as H
    return sum(r.send.size for r in regions if H.neighbor(cfg, rank, r.dir) != rank)


def _reduce(torch, world, v, op):
    if world == 1:
        return v
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cpu" if dist.get_backend() == "gloo" else "cuda")
    dist.all_reduce(t, op=op)
    return float(t.item())


def halo_section(torch, rank, world, local, job, iters=20, warmup=5, nccl=True):
    import paper_2012_14363_b200.halo as H
    import paper_2012_14363_b200.rt as rt
    import torch.distributed as dist
    grid = GRIDS.get(world)
    if grid is None:
        return {"skipped": f"no 3D grid for {world} ranks"}
    cfg = H.HaloConfig(grid, (256, 256, 256), 2, 32)
    regions = H.build_halo_types(cfg)
    ndev = torch.cuda.device_count()
    if world > 1 and ndev > 1:
        nv = nvlink_peak(torch, local, (local + 1) % ndev)
        nv_src = f"measured in this run: cudaMemcpyPeerAsync cuda:{local} -> cuda:{(local + 1) % ndev}"
    else:
        nv, nv_src = NVLINK_FALLBACK_GBPS, "B200_PROFILING.md fallback (no peer GPU visible)"
    pad = 260 ** 3 * 32
    seg = [0]
    for r in regions:
        seg.append(seg[-1] + r.send.size)
    rt.init(rank, world, job, device=local, window_bytes=1 << 20, host_bytes=1 << 20)
    alloc = torch.empty(pad, dtype=torch.uint8, device="cuda")
    H.fill(cfg, rank, alloc)
    torch.cuda.synchronize()
    MAX = dist.ReduceOp.MAX if world > 1 else None

    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    sink = torch.empty(1, dtype=torch.int64, device="cuda")
    rt_stream = torch.cuda.ExternalStream(rt.stream())

    def cold(i, on=None):
        # 512 MiB written then read back ON THE PLAN'S STREAM, not waited
        # for: every timed exchange starts on a cold, clean L2 (the halo's
        # 51 MB would otherwise stay L2-resident between iterations, which a
        # stencil sweep in between would not allow), and its start event is
        # reached only after the exchange's launches are enqueued, so host
        # launch latency is not timed
        with torch.cuda.stream(on if on is not None else rt_stream):
            flush.fill_(i & 0xFF)
            torch.sum(flush.view(torch.int64), dim=0, out=sink[0])

    def run(method):
        H.fill(cfg, rank, alloc)
        torch.cuda.synchronize()
        plan = rt.HaloPlan(cfg, alloc, method)
        for i in range(warmup):
            cold(i)
            plan.exchange()
        ts = []
        for i in range(iters):
            cold(i)
            ts.append(plan.exchange())
        bad = H.verify(cfg, rank, alloc)
        plan.free()
        ph = {k: _reduce(torch, world, statistics.median(t[k] for t in ts), MAX) for k in ts[0]}
        return ph, _reduce(torch, world, float(bad), MAX)

    phase_direct, bad_direct = run(H.DIRECT)  # ghost writes: one typed-copy launch, no packed segments
    phase, bad = run(H.FUSED_ASYNC)      # device-ordered: completion flags, no host barrier
    phase_sync, bad_sync = run(H.FUSED)  # host-barrier variant, for comparison
    bad = max(bad, bad_sync, bad_direct)
    rbytes = remote_bytes(cfg, regions, rank)
    out = {"grid": list(grid), "interior": 256, "radius": 2, "element_bytes": 32,
           "l2": "flushed (512 MiB write + read, enqueued on the plan's stream) before every exchange",
           "bytes_per_rank": seg[-1], "remote_bytes_per_rank": rbytes, "verified": bad == 0,
           "direct_us": {"iteration": round(phase_direct["iteration"] * 1e6, 2),
                         "how": "one typed-copy launch per rank writes every ghost region in place "
                                "(in-kernel completion flags to remote neighbours)"},
           "direct_hbm_GBps_per_rank": round(2 * seg[-1] / phase_direct["iteration"] / 1e9, 1),
           "direct_hbm_frac": round(2 * seg[-1] / phase_direct["iteration"] / 1e9 / _hbm_peak(), 3),
           "direct_frac_of_nvlink_bound": (round(rbytes / (nv * 1e9) / phase_direct["iteration"], 3)
                                           if rbytes else None),
           "nvlink_peak_GBps": round(nv, 1), "nvlink_peak_source": nv_src,
           "fused_us": {k: round(v * 1e6, 2) for k, v in phase.items()},
           "fused_hostsync_us": {k: round(v * 1e6, 2) for k, v in phase_sync.items()},
           "fused_hbm_GBps_per_rank": round(4 * seg[-1] / phase["iteration"] / 1e9, 1),
           "nvlink_bound_us": round(rbytes / (nv * 1e9) * 1e6, 2)}
    # the same exchange through the MPI-level call (MPI_Neighbor_alltoallw
    # with the 26 region types): one typed-copy launch per rank plus the
    # per-call entry protocol and a stream synchronisation; wall time
    import time
    H.fill(cfg, rank, alloc)
    torch.cuda.synchronize()
    sends = [(H.neighbor(cfg, rank, r.dir), 1, r.send, 0) for r in regions]
    recvs = [(H.neighbor(cfg, rank, tuple(-x for x in r.dir)), 1, regions[25 - j].recv, 0)
             for j, r in enumerate(regions)]
    nw = rt.NeighborW(sends, recvs)
    ws = []
    for i in range(warmup + iters):
        cold(i)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        nw(alloc, alloc)
        if i >= warmup:
            ws.append(time.perf_counter() - t0)
    bad_w = H.verify(cfg, rank, alloc)
    out["mpi_alltoallw_us"] = round(_reduce(torch, world, statistics.median(ws), MAX) * 1e6, 2)
    # the same as an MPI-4 persistent collective (compiled once; a start is
    # one signalled launch, no host entry protocol): start + wait, wall time
    try:
        plan = rt.NeighborPlan(sends, recvs, alloc, alloc)
        H.fill(cfg, rank, alloc)
        torch.cuda.synchronize()
        ps = []
        for i in range(warmup + iters):
            cold(i)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            plan.start()
            plan.wait()
            if i >= warmup:
                ps.append(time.perf_counter() - t0)
        bad_w += H.verify(cfg, rank, alloc)
        plan.free()
        out["mpi_alltoallw_persistent_us"] = round(_reduce(torch, world, statistics.median(ps), MAX) * 1e6, 2)
    except Exception as exc:
        out["mpi_alltoallw_persistent_us"] = {"error": f"{type(exc).__name__}: {exc}"}
    out["verified"] = out["verified"] and _reduce(torch, world, float(bad_w), MAX) == 0
    if nccl and world > 1 and dist.is_initialized() and dist.get_backend() == "nccl":
        out["nccl"] = _nccl_halo(torch, cfg, regions, seg, alloc, rank, world, iters, warmup, cold)
    try:  # an optional row: its failure must not cost the measured ones above
        out["steady_state"] = _halo_steady(torch, rt, H, cfg, alloc, rank, world)
    except Exception as exc:
        out["steady_state"] = {"error": f"{type(exc).__name__}: {exc}"}
    rt.finalize()
    return out


def _halo_steady(torch, rt, H, cfg, alloc, rank, world, iters=200, per_graph=10):
    """the iterations of a time loop: exchanges back to back with no host
    synchronisation and no L2 flush between them, enqueued eagerly, or
    replayed from a CUDA graph holding `per_graph` exchanges (the plan then
    numbers its iterations on the device). Wall time per iteration over
    `iters` iterations, max over ranks; every ghost verified after a
    replay."""
    import time
    import paper_2012_14363_b200 as sp
    import torch.distributed as dist
    MAX = dist.ReduceOp.MAX if dist.is_initialized() else None
    rs = torch.cuda.ExternalStream(rt.stream())
    out = {"how": f"{iters} back-to-back exchanges, warm L2, wall time per iteration (max over ranks); "
                  f"graph = replays of a CUDA graph of {per_graph} exchanges"}
    for method, name in ((H.DIRECT, "direct"), (H.FUSED_ASYNC, "fused_async")):
        H.fill(cfg, rank, alloc)
        torch.cuda.synchronize()
        rt.barrier()
        plan = rt.HaloPlan(cfg, alloc, method)
        for _ in range(5):
            plan.exchange(timed=False)
        rs.synchronize()
        rt.barrier()
        t0 = time.perf_counter()
        for _ in range(iters):
            plan.exchange(timed=False)
        rs.synchronize()
        eager = _reduce(torch, world, (time.perf_counter() - t0) / iters, MAX)
        row = {"eager_us": round(eager * 1e6, 2)}
        g = torch.cuda.CUDAGraph()
        refused = False
        with torch.cuda.stream(rs):
            g.capture_begin()
            try:
                for _ in range(per_graph):
                    plan.exchange(timed=False)
            except sp.Unsupported:
                refused = True
            finally:
                g.capture_end()
        if refused:
            row["graph"] = "refused"
        else:
            with torch.cuda.stream(rs):
                g.replay()
            rs.synchronize()
            rt.barrier()
            t0 = time.perf_counter()
            with torch.cuda.stream(rs):
                for _ in range(iters // per_graph):
                    g.replay()
            rs.synchronize()
            graph = _reduce(torch, world, (time.perf_counter() - t0) / iters, MAX)
            H.fill(cfg, rank, alloc)
            torch.cuda.synchronize()
            rt.barrier()
            with torch.cuda.stream(rs):
                g.replay()
            rs.synchronize()
            bad = _reduce(torch, world, float(H.verify(cfg, rank, alloc)), MAX)
            row.update({"graph_us": round(graph * 1e6, 2), "speedup": round(eager / graph, 2),
                        "verified": bad == 0})
        del g
        plan.free()
        out[name] = row
    return out


def _nccl_halo(torch, cfg, regions, seg, alloc, rank, world, iters, warmup, cold):
    """baseline: batch pack -> 26 NCCL send/recv in one group -> batch unpack"""
    import paper_2012_14363_b200.halo as H
    import torch.distributed as dist
    H.fill(cfg, rank, alloc)
    sbuf = torch.empty(seg[-1], dtype=torch.uint8, device="cuda")
    rbuf = torch.empty(seg[-1], dtype=torch.uint8, device="cuda")
    pack = H.Batch([(alloc, r.send, 1, sbuf, seg[j]) for j, r in enumerate(regions)])
    unpack = H.Batch([(rbuf, r.recv, 1, alloc, seg[k]) for k, r in enumerate(regions)], unpack=True)
    ops = []
    for j, r in enumerate(regions):
        ops.append(dist.P2POp(dist.isend, sbuf[seg[j]:seg[j + 1]], H.neighbor(cfg, rank, r.dir)))
    for k in range(25, -1, -1):  # the i-th recv from a peer matches its i-th send
        peer = H.neighbor(cfg, rank, regions[k].dir)
        ops.append(dist.P2POp(dist.irecv, rbuf[seg[k]:seg[k + 1]], peer))
    s = torch.cuda.current_stream()
    times = []
    for it in range(warmup + iters):
        dist.barrier()
        cold(it, s)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(s)
        pack.execute(s)
        ev[1].record(s)
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        ev[2].record(s)
        unpack.execute(s)
        ev[3].record(s)
        torch.cuda.synchronize()
        if it >= warmup:
            times.append([ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]),
                          ev[0].elapsed_time(ev[3])])
    bad = H.verify(cfg, rank, alloc)
    MAX = dist.ReduceOp.MAX
    med = [_reduce(torch, world, statistics.median(t[i] for t in times), MAX) for i in range(4)]
    return {"verified": _reduce(torch, world, float(bad), MAX) == 0,
            "us": {"pack": round(med[0] * 1e3, 2), "exchange": round(med[1] * 1e3, 2),
                   "unpack": round(med[2] * 1e3, 2), "iteration": round(med[3] * 1e3, 2)}}


def cfg4_prog(e0, n):
    """3D subarray with E0-byte blocks, n bytes total (BASELINE config 4):
    E1*E2 = n/E0 split as powers of two, sizes {max(2E0,64), 2E1, E2}."""
    rows = n // e0
    e2 = 2 ** (int(math.log2(rows)) // 2)
    e1 = rows // e2
    sizes = [max(2 * e0, 64), 2 * e1, e2]
    return [4, 3, 0] + sizes + [e0, e1, e2] + [0, 0, 0] + [0, 0]


def send_section(torch, rank, world, local, job, reps=10, warmup=3):
    """rank 0 -> rank 1, every method + model; other ranks idle"""
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.model as M
    import paper_2012_14363_b200.rt as rt
    if world < 2:
        return {"skipped": "needs 2 ranks"}
    rt.init(rank, world, job + "s", device=local, window_bytes=72 << 20, host_bytes=72 << 20)
    prof_path = os.path.join(ROOT, "profiles", "b200.profile")
    prof = M.load_profile_file(prof_path) if os.path.exists(prof_path) else None
    nv, nv_src, calib = NVLINK_FALLBACK_GBPS, "B200_PROFILING.md fallback", None
    if rank <= 1:
        other = 1 - rank  # rank r runs on device r (LOCAL_RANK)
        if torch.cuda.device_count() > 1 and local != other:
            nv = nvlink_peak(torch, local, other)
            nv_src = f"measured in this run: cudaMemcpyPeerAsync cuda:{local} -> cuda:{other}"
            if prof is not None:  # the model's peer terms, measured on this box before the sweep
                calib = calibrate_peer(torch, prof, local, other)
    if prof is not None:
        rt.set_profile(prof)
    rt.barrier()
    rows = []
    import time
    for e0 in (8, 64, 512):
        for n in [1 << k for k in range(10, 27, 4)]:
            if n < e0 * 4:
                continue
            ct = sp.commit_type(sp.from_program(cfg4_prog(e0, n)))
            buf = torch.zeros(ct.span, dtype=torch.uint8, device="cuda")
            row = {"E0": e0, "bytes": ct.size}
            for name, m in (("device", rt.DEVICE), ("oneshot", rt.ONESHOT), ("staged", rt.STAGED),
                            ("direct", rt.DIRECT), ("model", rt.AUTO)):
                ts, used = [], None
                for it in range(warmup + reps):
                    rt.barrier()
                    t0 = time.perf_counter()
                    if rank == 0:
                        used = rt.send(buf, 1, ct, 1, tag=it, method=m)
                        rt.recv(buf, 1, ct, source=1, tag=it)
                    elif rank == 1:
                        st = rt.recv(buf, 1, ct, source=0, tag=it)
                        used = st["method"]
                        rt.send(buf, 1, ct, 0, tag=it, method=m)
                    if it >= warmup:
                        ts.append((time.perf_counter() - t0) / 2)
                if rank <= 1:
                    row[name + "_us"] = round(statistics.median(ts) * 1e6, 2)
                    row[name + "_frac_of_nvlink"] = round(ct.size / statistics.median(ts) / 1e9 / nv, 3)
                    row[name + "_GBps"] = round(ct.size / statistics.median(ts) / 1e9, 2)
                    if name == "model":
                        row["model_choice"] = {0: "oneshot", 1: "device", 2: "staged", 3: "direct"}[used]
                        row["model_frac_of_nvlink"] = round(ct.size / statistics.median(ts) / 1e9 / nv, 3)
            rows.append(row)
    rt.finalize()
    _model_vs_fastest(rows)
    return {"pair": [0, 1], "timing": "half ping-pong wall time (host-synchronous MPI_Send/Recv semantics)",
            "nvlink_peak_GBps": round(nv, 1), "nvlink_peak_source": nv_src,
            "peer_calibration": calib, "checks": _checks(rows), "rows": rows}


def _checks(rows):
    """the send section's own consistency checks: the model within 10% of
    the fastest fixed method on every row, and STAGED (device pack + D2H +
    H2D + unpack) no slower than 1.3x ONE-SHOT at 64 MiB"""
    big = [r for r in rows if r["bytes"] >= (64 << 20) and "staged_us" in r and "oneshot_us" in r]
    return {"model_within_10pct_of_fastest": all(r.get("model_vs_fastest", 1.0) <= 1.10 for r in rows),
            "model_worst_vs_fastest": max((r.get("model_vs_fastest", 1.0) for r in rows), default=None),
            "staged_le_1.3x_oneshot_at_64MiB": all(r["staged_us"] <= 1.3 * r["oneshot_us"] for r in big),
            "staged_over_oneshot_at_64MiB": [round(r["staged_us"] / r["oneshot_us"], 3) for r in big]}


def _model_vs_fastest(rows):
    """the model's choice against the fastest fixed method of each row"""
    for row in rows:
        fixed = {k[:-3]: v for k, v in row.items() if k.endswith("_us") and k[:-3] in
                 ("device", "oneshot", "staged", "direct")}
        if fixed and "model_us" in row:
            best = min(fixed, key=fixed.get)
            row["fastest_fixed"] = best
            row["model_vs_fastest"] = round(row["model_us"] / fixed[best], 3)


def send_self_section(torch, rank, local, job, reps=7, warmup=2):
    """Config 4's code path on ONE GPU: rank 0 sends to itself (MPI_Isend +
    MPI_Irecv + MPI_Wait x2) with every method, 1 KiB - 64 MiB, E0 in
    {8, 64, 512}. No NVLink is involved: this measures the protocol, the
    kernels and the HBM traffic of each method (DEVICE = pack to the window +
    unpack, DIRECT = one typed copy, ONE-SHOT / STAGED over PCIe). Wall time
    per message, device buffers, L2 flushed before every message."""
    import time
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.model as M
    import paper_2012_14363_b200.rt as rt
    if rank != 0:
        return None
    rt.init(0, 1, job + "self", device=local, window_bytes=72 << 20, host_bytes=72 << 20)
    prof_path = os.path.join(ROOT, "profiles", "b200.profile")
    if os.path.exists(prof_path):
        rt.set_profile(M.load_profile_file(prof_path))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rows = []
    names = {0: "oneshot", 1: "device", 2: "staged", 3: "direct"}
    for e0 in (8, 64, 512):
        for n in [1 << k for k in range(10, 27, 4)]:
            if n < e0 * 4:
                continue
            ct = sp.commit_type(sp.from_program(cfg4_prog(e0, n)))
            src = torch.ones(ct.span, dtype=torch.uint8, device="cuda")
            dst = torch.zeros(ct.span, dtype=torch.uint8, device="cuda")
            row = {"E0": e0, "bytes": ct.size}
            for name, m in (("device", rt.DEVICE), ("direct", rt.DIRECT), ("oneshot", rt.ONESHOT),
                            ("staged", rt.STAGED), ("model", rt.AUTO)):
                ts, used = [], None
                for it in range(warmup + reps):
                    flush.fill_(it & 0xFF)
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    r = rt.irecv(dst, 1, ct, source=0, tag=it)
                    q = rt.isend(src, 1, ct, 0, tag=it, method=m)
                    q.wait()
                    used = r.wait()["method"]
                    if it >= warmup:
                        ts.append(time.perf_counter() - t0)
                t = statistics.median(ts)
                row[name + "_us"] = round(t * 1e6, 2)
                row[name + "_GBps"] = round(ct.size / t / 1e9, 2)
                if name == "model":
                    row["model_choice"] = names[used]
            rows.append(row)
    rt.finalize()
    _model_vs_fastest(rows)
    return {"pair": [0, 0], "timing": "wall time of Isend+Irecv+Wait to self, median; device buffers; "
                                      "one GPU (no NVLink): protocol + kernels + HBM/PCIe traffic per method",
            "checks": _checks(rows), "rows": rows}


if __name__ == "__main__":  # one-rank halo section alone: python tools/bench_parts.py
    import json
    import uuid

    import torch
    torch.cuda.set_device(0)
    print(json.dumps(halo_section(torch, 0, 1, 0, uuid.uuid4().hex[:10])))


def irregular_section(torch, blocks=(64, 1024, 4096), total=64 << 20, reps=5):
    """Beyond the reference: irregular MPI_Type_create_hindexed byte types of
    ~64 MiB (blocks of L/2..3L/2 bytes in multiples of 16 at random 16-B
    gaps, scrambled definition order) through the run-table kernel, against
    the regular hvector of the same mean block and pitch on the strided
    kernels. Cold L2 (512 MiB flush on the timing stream), CUDA events,
    median of `reps`; GB/s = 2 x packed bytes / kernel time."""
    import numpy as np
    import paper_2012_14363_b200 as sp
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    B = sp.make_named(sp.NamedKind.Byte)
    rng = np.random.default_rng(1)

    def timed(fn):
        ts = []
        for _ in range(reps):
            flush.fill_(1)  # 512 MiB written, then read back: a cold, clean L2
            flush.view(torch.int64).sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        return statistics.median(ts)

    rows = []
    for L in blocks:
        n = total // L
        lens = (rng.integers(L // 32, 3 * L // 32 + 1, n).clip(1) * 16).astype(np.int64)
        gaps = (rng.integers(0, L // 16 + 1, n) * 16).astype(np.int64)
        displs = np.cumsum(gaps + lens) - lens
        perm = rng.permutation(n)
        t = sp.commit_type(sp.make_hindexed(lens[perm].tolist(), displs[perm].tolist(), B))
        src = torch.randint(0, 256, (t.span,), dtype=torch.uint8, device="cuda")
        dst = torch.empty(t.size, dtype=torch.uint8, device="cuda")
        pitch = max(int(np.mean(gaps + lens)) // 16 * 16, L)
        v = sp.commit_type(sp.make_hvector(total // L, L, pitch, B))
        vsrc = torch.randint(0, 256, (v.span,), dtype=torch.uint8, device="cuda")
        vdst = torch.empty(v.size, dtype=torch.uint8, device="cuda")
        pk = timed(lambda: sp.pack(src, t, 1, dst, 0))
        li = sp.last_launch()
        up = timed(lambda: sp.unpack(dst, 0, t, 1, src))
        vp = timed(lambda: sp.pack(vsrc, v, 1, vdst, 0))
        vu = timed(lambda: sp.unpack(vdst, 0, v, 1, vsrc))
        rows.append({"mean_block": L, "runs": int(n), "bytes": int(t.size),
                     "kernel": f"{li.kernel.name}/w{li.word}",
                     "pack_GBps": round(2 * t.size / pk / 1e3, 1), "unpack_GBps": round(2 * t.size / up / 1e3, 1),
                     "pack_frac_of_hbm": round(2 * t.size / pk / 1e3 / _hbm_peak(), 3),
                     "strided_pack_GBps": round(2 * v.size / vp / 1e3, 1),
                     "strided_unpack_GBps": round(2 * v.size / vu / 1e3, 1)})
        del src, dst, vsrc, vdst
    del flush
    torch.cuda.empty_cache()
    return {"what": "irregular hindexed types (beyond the reference) on the run-table kernel vs the regular "
                    "hvector of the same mean block and pitch on the strided kernels; cold L2",
            "rows": rows}


def interpose_section(timeout_s=240.0, budget_s=2.0):
    """TEMPI as a PMPI interposer over a system MPI: two
    portable MPI programs on the stand-in system MPI (tests/native/minimpi.c:
    a CUDA-aware MPI whose device derived types move one cudaMemcpy per
    contiguous run, the generic path) alone, then the same binaries with
    LD_PRELOAD=libtempi_interpose.so. 2 ranks on this GPU.
      * tools/interpose_bench.c: MPI_Pack / MPI_Unpack of the cfg1 vector and
        cfg2 subarrays (E0 = 64, 512) on device memory, MPI_Send/Recv of the
        cfg1 object;
      * tests/native/mpi_halo.c: the config-5 halo (256^3, r = 2, 32 B) on
        one rank (periodic: all 26 neighbours are the rank itself; two
        processes on one GPU would time-slice) as MPI_Pack x26 +
        MPI_Neighbor_alltoallv (MPI_PACKED, forwarded in both legs) +
        MPI_Unpack x26, and as one MPI_Neighbor_alltoallw of the region
        types; every ghost cell verified.
    Returns {case: {bytes, system_mpi_us, tempi_us, speedup}}."""
    import json
    import re
    import subprocess
    import tempfile

    pkg = os.path.join(ROOT, "paper_2012_14363_b200")
    inc = ["-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include"]
    cuda = "/usr/local/cuda/lib64"
    legs = {"system_mpi": {}, "tempi": {}}
    with tempfile.TemporaryDirectory() as d:
        lib = os.path.join(d, "libminimpi.so")
        subprocess.run(["/usr/bin/gcc", "-O2", "-fPIC", "-shared", "-pthread"] + inc +
                       [os.path.join(ROOT, "tests", "native", "minimpi.c"), "-o", lib, "-L" + cuda, "-lcudart",
                        "-Wl,-rpath," + cuda], check=True)
        exes = {}
        for name, src in (("interpose_bench", os.path.join(ROOT, "tools", "interpose_bench.c")),
                          ("mpi_halo", os.path.join(ROOT, "tests", "native", "mpi_halo.c"))):
            exes[name] = os.path.join(d, name)
            subprocess.run(["/usr/bin/gcc", "-O2"] + inc + [src, "-o", exes[name], "-L" + d, "-lminimpi",
                            "-L" + pkg, "-lstridepack_b200", "-L" + cuda, "-lcudart", "-Wl,-rpath," + d,
                            "-Wl,-rpath," + pkg, "-Wl,-rpath," + cuda], check=True)

        def launch(leg, args, n=2):
            env = dict(os.environ)
            if leg == "tempi":
                env["LD_PRELOAD"] = os.path.join(pkg, "libtempi_interpose.so")
            p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "tempirun.py"), "-n", str(n), "--timeout",
                                str(timeout_s)] + args, capture_output=True, text=True, env=env,
                               timeout=timeout_s + 30)
            if p.returncode != 0:
                raise RuntimeError(f"{leg} {os.path.basename(args[0])}: rc {p.returncode}: "
                                   f"{p.stdout[-300:]} {p.stderr[-300:]}")
            return p.stdout

        for leg in legs:
            out = launch(leg, [exes["interpose_bench"], str(budget_s)])
            legs[leg] = {r["what"]: r for r in map(json.loads, filter(None, out.splitlines()))}
            for mode in (0, 1):
                out = launch(leg, [exes["mpi_halo"], "1", "1", "1", "256", "2", "32", "2", str(mode)], n=1)
                m = re.search(r"pack ([\d.]+) us alltoallv ([\d.]+) us unpack ([\d.]+) us bytes/rank (\d+)", out)
                if not m or "OK" not in out:
                    raise RuntimeError(f"{leg} mpi_halo mode {mode}: {out[-300:]}")
                tp, tx, tu, nb = float(m[1]), float(m[2]), float(m[3]), int(m[4])
                if mode == 0:
                    legs[leg]["halo 1x1x1 MPI_Pack x26"] = {"bytes": nb, "us": tp}
                    legs[leg]["halo 1x1x1 MPI_Neighbor_alltoallv (MPI_PACKED)"] = {"bytes": nb, "us": tx}
                    legs[leg]["halo 1x1x1 MPI_Unpack x26"] = {"bytes": nb, "us": tu}
                else:
                    legs[leg]["halo 1x1x1 MPI_Neighbor_alltoallw (26 region types)"] = {"bytes": nb, "us": tx}
    out = {}
    for what, r in legs["tempi"].items():
        s = legs["system_mpi"].get(what)
        out[what] = {"bytes": r["bytes"], "system_mpi_us": s["us"] if s else None, "tempi_us": r["us"],
                     "speedup": round(s["us"] / r["us"], 1) if s and r["us"] > 0 else None}
    return {"how": "same binaries with and without LD_PRELOAD=libtempi_interpose.so; system MPI = "
                   "tests/native/minimpi.c (contiguous data in one cudaMemcpy; device derived types one "
                   "cudaMemcpy per contiguous run on the device, then one copy to or from its host message "
                   "buffer; socket transport); "
                   "tools/interpose_bench.c on 2 ranks (rank 0 packs; Send/Recv 0 -> 1): best of <=5 warm "
                   "calls; tests/native/mpi_halo.c 1x1x1 256^3 r=2 32 B on 1 rank: wall time of the second of "
                   "2 iterations, every ghost cell verified",
            "cases": out}
