"""Unstructured-mesh style neighbour exchange on one rank (every edge to
itself): 26 irregular MPI_Type_indexed gather lists of doubles (blocks of
1-4 doubles at scrambled slots of a 4M-double field), contiguous ghost
receive runs. Wall time per MPI_Neighbor_alltoallw call (all 26 irregular
edges packed by ONE k_runs_multi launch, then a stream sync) against the
same 26 gathers as 26 separate sp.pack launches + one sync; then the
reverse (scattered ghosts): contiguous sends scattered through the 26
irregular types as receive layouts. Median of 50, warm."""
import json
import statistics
import sys
import time
import uuid

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2012_14363_b200 as sp  # noqa: E402
import paper_2012_14363_b200.rt as rt  # noqa: E402

torch.cuda.set_device(0)
rt.init(0, 1, "uh" + uuid.uuid4().hex[:8], device=0, window_bytes=1 << 20, host_bytes=1 << 20)
D = sp.make_named(sp.NamedKind.Double)
rng = np.random.default_rng(3)
N = 4 << 20
out = {}
for nblocks in (500, 5000):
    types, sizes = [], []
    disjoint = rng.permutation(N // 4)  # the edges' slot sets do not overlap (ghosts of distinct neighbours)
    for e in range(26):
        bl = rng.integers(1, 5, nblocks).tolist()
        slots = disjoint[e * nblocks:(e + 1) * nblocks]
        t = sp.commit_type(sp.make_indexed(bl, [int(x) * 4 for x in slots], D))
        types.append(t)
        sizes.append(sum(bl))
    ghosts = [sp.commit_type(sp.make_contiguous(n, D)) for n in sizes]
    field = torch.randn(N, dtype=torch.float64, device="cuda")
    recv = torch.empty(sum(sizes), dtype=torch.float64, device="cuda")
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]) * 8
    call = rt.NeighborW([(0, 1, t, 0) for t in types], [(0, 1, g, int(o)) for g, o in zip(ghosts, offs)])
    for _ in range(5):
        call(field, recv)
    ws = []
    for _ in range(50):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        call(field, recv)
        ws.append(time.perf_counter() - t0)
    # correctness spot check: edge 0
    ref = torch.empty(sizes[0], dtype=torch.float64, device="cuda")
    sp.pack(field, types[0], 1, ref, 0)
    assert torch.equal(ref, recv[:sizes[0]])
    ps = []
    for _ in range(50):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for t, o in zip(types, offs):
            sp.pack(field, t, 1, recv.view(torch.uint8)[int(o):], 0)
        torch.cuda.synchronize()
        ps.append(time.perf_counter() - t0)
    # scattered ghosts: contiguous sends, the 26 irregular types as RECEIVE
    # layouts (the sender scatters through the receiver's run table)
    flat = torch.randn(sum(sizes), dtype=torch.float64, device="cuda")
    ghost_field = torch.zeros(N, dtype=torch.float64, device="cuda")
    call2 = rt.NeighborW([(0, 1, g, int(o)) for g, o in zip(ghosts, offs)], [(0, 1, t, 0) for t in types])
    try:
        call2(flat, ghost_field)
    except sp.Unsupported:  # irregular receive layouts are disabled in the engine
        out[nblocks] = {"bytes": int(sum(sizes) * 8), "alltoallw_us": round(statistics.median(ws) * 1e6, 1),
                        "per_edge_packs_us": round(statistics.median(ps) * 1e6, 1)}
        print(json.dumps({nblocks: out[nblocks]}), flush=True)
        continue
    for _ in range(5):
        call2(flat, ghost_field)
    ws2 = []
    for _ in range(50):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        call2(flat, ghost_field)
        ws2.append(time.perf_counter() - t0)
    back = torch.empty(sizes[0], dtype=torch.float64, device="cuda")
    sp.pack(ghost_field, types[0], 1, back, 0)
    assert torch.equal(back, flat[:sizes[0]])
    out[nblocks] = {"bytes": int(sum(sizes) * 8), "alltoallw_us": round(statistics.median(ws) * 1e6, 1),
                    "per_edge_packs_us": round(statistics.median(ps) * 1e6, 1),
                    "scattered_ghosts_alltoallw_us": round(statistics.median(ws2) * 1e6, 1)}
    print(json.dumps({nblocks: out[nblocks]}), flush=True)
rt.finalize()
