"""3D halo exchange (H1): region geometry against the reference's own halo
types (tests/golden/halo_golden.json), the KATs of proj/tests/test_halo.cpp,
and on the GPU the full exchange (fused pack-to-peer batches and the copy
baseline) verified cell-for-cell with the reference's fill_cell pattern and
its modeled phase times reproduced exactly."""
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def H():
    import paper_2012_14363_b200.halo as h
    return h


@pytest.fixture(scope="module")
def hgold():
    return json.load(open(os.path.join(GOLD, "halo_golden.json")))


def test_region_types_match_reference(sp, H, orc, hgold):
    for g in hgold["types"]:
        cfg = H.HaloConfig(interior=tuple(g["interior"]), radius=g["radius"], element_bytes=g["elem"])
        regs = H.build_halo_types(cfg)
        assert len(regs) == 26
        for mine, ref in zip(regs, g["regions"]):
            assert list(mine.dir) == ref["dir"] and mine.gridpoints == ref["cells"]
            for ct, prog in ((mine.send, ref["send"]), (mine.recv, ref["recv"])):
                want = orc.commit(prog)
                assert (ct.size, ct.extent, ct.span, ct.overlapping) == (want.size, want.extent, want.span,
                                                                          want.overlapping)
                assert ct.canon == sp.StridedBlock(want.start, tuple(want.counts), tuple(want.strides))


def test_face_edge_corner_geometry(H):
    """test_halo.cpp:11-44"""
    cfg = H.HaloConfig(interior=(16, 16, 16), radius=3, element_bytes=64)
    regs = H.build_halo_types(cfg)
    faces = edges = corners = recv_cells = 0
    for r in regs:
        axes = sum(abs(x) for x in r.dir)
        want = {1: 3 * 16 * 16, 2: 3 * 3 * 16, 3: 27}[axes]
        assert r.gridpoints == want
        assert r.send.size == want * 64 and r.recv.size == want * 64
        faces += axes == 1
        edges += axes == 2
        corners += axes == 3
        recv_cells += r.gridpoints
    assert (faces, edges, corners) == (6, 12, 8)
    assert recv_cells == 22 ** 3 - 16 ** 3
    small = H.build_halo_types(H.HaloConfig(interior=(2, 2, 2), radius=1, element_bytes=8))
    assert all(r.gridpoints == 1 for r in small if sum(abs(x) for x in r.dir) == 3)


def test_config_validation(sp, H):
    """test_halo.cpp:58-68"""
    with pytest.raises(sp.InvalidArgument):
        H.build_halo_types(H.HaloConfig(interior=(4, 4, 4), radius=3))
    with pytest.raises(sp.InvalidArgument):
        H.build_halo_types(H.HaloConfig(interior=(4, 4, 4), radius=0))
    H.build_halo_types(H.HaloConfig(interior=(4, 4, 4), radius=2))
    with pytest.raises(sp.InvalidArgument):
        H.neighbor(H.HaloConfig(ranks=(0, 1, 1), interior=(4, 4, 4), radius=2), 0, (1, 0, 0))


def test_neighbor_mapping(H):
    cfg = H.HaloConfig(ranks=(3, 1, 2), interior=(4, 6, 8), radius=2)
    # rank = (z*R1 + y)*R0 + x, periodic
    assert H.neighbor(cfg, 0, (-1, 0, 0)) == 2
    assert H.neighbor(cfg, 0, (0, 0, 1)) == 3
    assert H.neighbor(cfg, 5, (1, 1, 1)) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("method", [0, 1, 3])
def test_exchange_matches_reference_reports(H, cuda, hgold, method):
    """run_exchange: every ghost cell exact; bytes moved and the modeled
    phase times equal the reference's ExchangeReport (halo.hpp:287-320)."""
    import paper_2012_14363_b200.model as M
    prof = M.load_profile_file(os.path.join(GOLD, "default.profile"))
    for r in hgold["reports"]:
        cfg = H.HaloConfig(tuple(r["ranks"]), tuple(r["interior"]), r["radius"], r["elem"])
        rep = H.run_exchange(cfg, prof, method=method, iters=2)
        assert rep.verified and rep.mismatched_cells == 0, r
        assert rep.bytes_moved == r["bytes"]
        assert (rep.pack_seconds, rep.alltoallv_seconds, rep.unpack_seconds) == (r["pack"], r["alltoallv"],
                                                                                 r["unpack"])
        assert rep.measured_pack_seconds > 0
        assert rep.measured_unpack_seconds > 0 or method == H.DIRECT  # DIRECT has no unpack phase


@pytest.mark.gpu
def test_randomized_desk_scale_exchanges(H, cuda):
    """test_halo.cpp:108-125"""
    rng = np.random.default_rng(314)
    for _ in range(6):
        radius = 1 + int(rng.integers(0, 2))
        ranks = tuple(1 + int(rng.integers(0, 3)) for _ in range(3))
        interior = tuple(2 * radius + int(rng.integers(0, 8)) for _ in range(3))
        elem = [1, 4, 8, 64][int(rng.integers(0, 4))]
        for method in (0, 1, 3):
            rep = H.run_exchange(H.HaloConfig(ranks, interior, radius, elem), None, method=method)
            assert rep.verified, (ranks, interior, radius, elem, method)


@pytest.mark.gpu
def test_verify_detects_unexchanged_ghosts(H, cuda):
    torch = cuda
    cfg = H.HaloConfig((1, 1, 1), (6, 6, 6), 1, 8)
    alloc = torch.empty(8 ** 3 * 8, dtype=torch.uint8, device="cuda")
    H.fill(cfg, 0, alloc)
    assert H.verify(cfg, 0, alloc) == 8 ** 3 - 6 ** 3  # every ghost cell is still 0xee
    host = alloc.cpu().numpy().reshape(8, 8, 8, 8)
    assert (host[0, 0, 0] == 0xEE).all() and not (host[1, 1, 1] == 0xEE).all()


@pytest.mark.gpu
def test_batch_parity_vs_oracle(sp, orc, cuda, corpus):
    """many (type, buffer) jobs in one launch == per-job oracle packs"""
    torch = cuda
    from paper_2012_14363_b200.halo import Batch
    rng = np.random.default_rng(9)
    picks = [e for e in corpus if e["ref"]["status"] == 0 and e["ref"]["form"] == 0
             and 0 < e["ref"]["size"] <= (1 << 14)][:120]
    jobs, wants, srcs = [], [], []
    total = sum(e["ref"]["size"] * 2 for e in picks) + 16 * len(picks)
    packed = torch.zeros(total, dtype=torch.uint8, device="cuda")
    pos = 0
    for e in picks:
        ct = sp.commit_type(sp.from_program(e["prog"]))
        inc = 1 + int(rng.integers(0, 2))
        span = (inc - 1) * ct.extent + ct.span
        host = rng.integers(0, 256, span, dtype=np.uint8)
        src = torch.from_numpy(host).cuda()
        srcs.append(src)
        want = np.zeros(inc * ct.size, np.uint8)
        assert orc.pack(e["prog"], host, inc, want, 0)[0] == 0
        jobs.append((src, ct, inc, packed, pos))
        wants.append((pos, want, e["prog"], inc, span, ct))
        pos += inc * ct.size + int(rng.integers(0, 3))
    b = Batch(jobs)
    assert b.bytes == sum(len(w[1]) for w in wants)
    b.execute()
    torch.cuda.synchronize()
    got = packed.cpu().numpy()
    for p, want, prog, inc, span, ct in wants:
        assert np.array_equal(got[p:p + len(want)], want), prog
    # unpack batch back into sentinel-filled buffers
    outs, ujobs = [], []
    for (p, want, prog, inc, span, ct) in wants:
        if ct.overlapping:
            continue
        o = torch.full((span,), 0x3C, dtype=torch.uint8, device="cuda")
        outs.append((o, p, want, prog, inc, span))
        ujobs.append((packed, ct, inc, o, p))
    Batch(ujobs, unpack=True).execute()
    torch.cuda.synchronize()
    for o, p, want, prog, inc, span in outs:
        exp = np.full(span, 0x3C, np.uint8)
        assert orc.unpack(prog, want, 0, inc, exp)[0] == 0
        assert np.array_equal(o.cpu().numpy(), exp), prog


def _pairs_of_equal_size(corpus, limit):
    """(A, B) corpus definitions describing the same byte count, B not
    self-overlapping: a typed copy A -> B is defined for them"""
    by_size = {}
    for e in corpus:
        r = e["ref"]
        if r["status"] == 0 and r["form"] == 0 and 0 < r["size"] <= (1 << 15):
            by_size.setdefault(r["size"], []).append(e)
    out = []
    for size, es in sorted(by_size.items()):
        for a in es:
            for b in es:
                if not b["ref"]["overlapping"] and len(out) < limit:
                    out.append((a, b))
    return out


@pytest.mark.gpu
def test_copy_batch_parity_vs_oracle(sp, orc, cuda, corpus):
    """typed copies A -> B in one launch == oracle unpack(B, oracle pack(A));
    bytes outside B's layout keep their sentinel"""
    torch = cuda
    from paper_2012_14363_b200.halo import Batch
    rng = np.random.default_rng(21)
    pairs = _pairs_of_equal_size(corpus, 150)
    assert len(pairs) >= 50
    jobs, checks = [], []
    for a, b in pairs:
        ca, cb = sp.commit_type(sp.from_program(a["prog"])), sp.commit_type(sp.from_program(b["prog"]))
        host = rng.integers(0, 256, ca.span, dtype=np.uint8)
        src = torch.from_numpy(host).cuda()
        dst = torch.full((cb.span + 7,), 0x5A, dtype=torch.uint8, device="cuda")
        packed = np.zeros(ca.size, np.uint8)
        assert orc.pack(a["prog"], host, 1, packed, 0)[0] == 0
        exp = np.full(cb.span + 7, 0x5A, np.uint8)
        assert orc.unpack(b["prog"], packed, 0, 1, exp)[0] == 0
        jobs.append((src, ca, 1, dst, cb, 1))
        checks.append((src, dst, exp, a["prog"], b["prog"]))
    bt = Batch.copies(jobs)
    assert bt.bytes == sum(j[1].size for j in jobs)
    bt.execute()
    torch.cuda.synchronize()
    for src, dst, exp, pa, pb in checks:
        assert np.array_equal(dst.cpu().numpy(), exp), (pa, pb)


@pytest.mark.gpu
def test_copy_batch_counts_and_errors(sp, orc, cuda):
    """count != 1 on either side (objects one extent apart), and the
    validation of sp_copy_batch_create"""
    torch = cuda
    from paper_2012_14363_b200.halo import Batch
    a = sp.commit_type(sp.make_vector(6, 2, 5, sp.make_named(sp.NamedKind.Int)))      # 48 B
    b = sp.commit_type(sp.make_hvector(4, 1, 40, sp.make_contiguous(12, sp.make_named(sp.NamedKind.Byte))))  # 48 B
    rng = np.random.default_rng(4)
    span_a = 3 * a.extent + a.span
    host = rng.integers(0, 256, span_a, dtype=np.uint8)
    src = torch.from_numpy(host).cuda()
    dst = torch.zeros(3 * b.extent + b.span, dtype=torch.uint8, device="cuda")
    Batch.copies([(src, a, 4, dst, b, 4)]).execute()
    torch.cuda.synchronize()
    pa = [2, 6, 2, 5, 0, 1]
    pb = [3, 4, 1, 40, 1, 12, 0, 0]
    packed = np.zeros(4 * 48, np.uint8)
    assert orc.pack(pa, host, 4, packed, 0)[0] == 0
    exp = np.zeros(dst.numel(), np.uint8)
    assert orc.unpack(pb, packed, 0, 4, exp)[0] == 0
    assert np.array_equal(dst.cpu().numpy(), exp)
    # the same copy as a single by-value launch (sp_copy)
    dst.zero_()
    sp.copy(src, a, 4, dst, b, 4, sync=True)
    assert np.array_equal(dst.cpu().numpy(), exp)
    assert sp.last_launch().kernel == sp.Kernel.Batch
    with pytest.raises(sp.InvalidArgument):
        sp.copy(src, a, 4, dst, b, 3)
    with pytest.raises(sp.InvalidArgument):
        Batch.copies([(src, a, 4, dst, b, 3)])
    ov = sp.commit_type(sp.make_hvector(2, 1, 2, sp.make_contiguous(4, sp.make_named(sp.NamedKind.Byte))))
    with pytest.raises(sp.OverlappingLayout):
        Batch.copies([(src, sp.commit_type(sp.make_contiguous(8, sp.make_named(sp.NamedKind.Byte))), 1, dst, ov, 1)])
    with pytest.raises(sp.BufferTooSmall):
        Batch.copies([(src[:10], a, 1, dst, b, 1)])


@pytest.mark.gpu
@pytest.mark.parametrize("method", [3, 2])  # DIRECT, FUSED_ASYNC
def test_halo_exchange_graph_capture_one_rank(sp, cuda, method):
    """a 1x1x1 plan has no peer flags: its exchange captures into a CUDA
    graph as is; each replay rewrites every ghost cell (the shell is reset
    between replays), and the plan stays usable eagerly afterwards"""
    import uuid
    torch = cuda
    import paper_2012_14363_b200.halo as H
    import paper_2012_14363_b200.rt as rt
    rt.init(0, 1, "cap" + uuid.uuid4().hex[:8], device=0, window_bytes=1 << 20, host_bytes=1 << 20)
    try:
        cfg = H.HaloConfig((1, 1, 1), (12, 10, 8), 2, 16)
        alloc = torch.zeros(16 * 14 * 12 * 16, dtype=torch.uint8, device="cuda")
        plan = rt.HaloPlan(cfg, alloc, method)
        plan.exchange()
        rs = torch.cuda.ExternalStream(rt.stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(rs):
            g.capture_begin()
            try:
                plan.exchange(timed=False)
            finally:
                g.capture_end()
        for _ in range(3):
            H.fill(cfg, 0, alloc)
            torch.cuda.synchronize()
            with torch.cuda.stream(rs):
                g.replay()
            rs.synchronize()
            assert H.verify(cfg, 0, alloc) == 0
        H.fill(cfg, 0, alloc)
        torch.cuda.synchronize()
        plan.exchange()
        assert H.verify(cfg, 0, alloc) == 0
        del g
        plan.free()
    finally:
        rt.finalize()
