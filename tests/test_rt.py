"""The node-local runtime under the MPI surface, exercised with real
processes. CPU: bootstrap, barriers and control messages (world 2 and 3).
GPU (two processes sharing cuda:0 through CUDA IPC, the same code path as
two NVLink peers): datatype Send/Recv with every transfer method, bit-exact
against the oracle, and the distributed halo exchange verified cell by
cell."""
import multiprocessing as mp
import os
import sys
import traceback
import uuid

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _spawn(target, world, *args, timeout=240):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    job = uuid.uuid4().hex[:12]
    ps = [ctx.Process(target=_entry, args=(target, r, world, job, q) + args) for r in range(world)]
    for p in ps:
        p.start()
    results = {}
    try:
        for _ in range(world):
            r, ok, payload = q.get(timeout=timeout)
            results[r] = (ok, payload)
    finally:
        for p in ps:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r in range(world):
        ok, payload = results[r]
        assert ok, f"rank {r}: {payload}"
    return {r: results[r][1] for r in range(world)}


def _entry(target, rank, world, job, q, *args):
    sys.path.insert(0, ROOT)
    try:
        q.put((rank, True, target(rank, world, job, *args)))
    except Exception:
        q.put((rank, False, traceback.format_exc()))


# ------------------------------------------------------------ CPU control plane
def _control(rank, world, job):
    import paper_2012_14363_b200.rt as rt
    rt.init(rank, world, job, device=-1)
    assert rt.rank() == rank and rt.size() == world
    for _ in range(200):
        rt.barrier()
    # ring of control messages, two laps, tags kept apart
    right, left = (rank + 1) % world, (rank - 1) % world
    rt.host_send(right, 7, f"r{rank}".encode())
    rt.host_send(right, 9, b"tag9")
    got9 = rt.host_recv(left, 9)
    got7 = rt.host_recv(left, 7)
    assert got7 == f"r{left}".encode() and got9 == b"tag9"
    rt.finalize()
    return "ok"


@pytest.mark.parametrize("world", [2, 3])
def test_runtime_control_plane(world):
    assert set(_spawn(_control, world).values()) == {"ok"}


def _dead_peer(rank, world, job):
    """rank 1 exits without finalising; rank 0's barrier notices the dead
    process and raises Timeout (long before TEMPI_TIMEOUT)"""
    import time
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.rt as rt
    rt.init(rank, world, job, device=-1)
    if rank == 1:
        os._exit(0)
    t0 = time.time()
    try:
        rt.barrier()
        return "no error"
    except sp.Timeout as e:
        return ("Timeout", "exited" in str(e), time.time() - t0 < 30)


def _stuck_peer(rank, world, job):
    """rank 1 is alive but never enters the barrier: rank 0 gives up after
    TEMPI_TIMEOUT seconds with Timeout"""
    import time
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.rt as rt
    rt.init(rank, world, job, device=-1)
    if rank == 1:
        time.sleep(6)
        return "slept"
    t0 = time.time()
    try:
        rt.barrier()
        return "no error"
    except sp.Timeout as e:
        return ("Timeout", "TEMPI_TIMEOUT" in str(e), 0.8 < time.time() - t0 < 5)


def _spawn_raw(target, world, want=None, timeout=60):
    """like _spawn, but only the ranks in `want` must report (a rank that
    exits without reporting is not an error)"""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    job = uuid.uuid4().hex[:12]
    ps = [ctx.Process(target=_entry, args=(target, r, world, job, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = {}
    want = set(range(world)) if want is None else set(want)
    try:
        while not want <= set(out):
            try:
                r, ok, payload = q.get(timeout=timeout)
            except Exception:
                break
            out[r] = payload if ok else "error: " + payload
    finally:
        for p in ps:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    return out


def test_runtime_dead_peer_raises_timeout():
    res = _spawn_raw(_dead_peer, 2, want=[0])
    assert res.get(0) == ("Timeout", True, True), res


def test_runtime_stuck_peer_times_out(monkeypatch):
    monkeypatch.setenv("TEMPI_TIMEOUT", "1")
    res = _spawn_raw(_stuck_peer, 2)
    assert res.get(0) == ("Timeout", True, True), res


# ------------------------------------------------------------ GPU data plane
def _sendrecv(rank, world, job):
    import torch
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.rt as rt
    import paper_2012_14363_b200.model as M
    from oracle.pyoracle import oracle
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=64 << 20, host_bytes=64 << 20)
    rt.set_profile(M.load_profile_file(os.path.join(ROOT, "tests", "golden", "default.profile")))
    # cfg4-shaped object: subarray block E0=64 at 1 KiB pitch, 3D
    prog = [4, 3, 0, 128, 64, 16, 64, 32, 8, 16, 8, 4, 0, 0]
    ct = sp.commit_type(sp.from_program(prog))
    out = []
    for i, method in enumerate([rt.DEVICE, rt.ONESHOT, rt.STAGED, rt.AUTO]):
        count = 1 + i % 2
        span = (count - 1) * ct.extent + ct.span
        rng = np.random.default_rng(100 + i)
        host = rng.integers(0, 256, span, dtype=np.uint8)
        if rank == 0:
            used = rt.send(torch.from_numpy(host).cuda(), count, ct, 1, tag=i, method=method)
            out.append(used)
        else:
            dst = torch.full((span,), 0x11, dtype=torch.uint8, device="cuda")
            st = rt.recv(dst, count, ct, source=0, tag=i)
            packed = np.zeros(count * ct.size, np.uint8)
            assert oracle().pack(prog, host, count, packed, 0)[0] == 0
            want = np.full(span, 0x11, np.uint8)
            assert oracle().unpack(prog, packed, 0, count, want)[0] == 0
            assert np.array_equal(dst.cpu().numpy(), want), (method, st)
            assert st["bytes"] == count * ct.size and st["source"] == 0 and st["tag"] == i
            out.append(st["method"])
    rt.finalize()
    return out


@pytest.mark.gpu
def test_sendrecv_every_method_two_processes(cuda):
    res = _spawn(_sendrecv, 2)
    assert res[0][:3] == [1, 0, 2] and res[1][:3] == [1, 0, 2]
    assert res[0][3] == res[1][3]  # the model's choice, seen identically on both sides


def _recv_buffer_too_small(rank, world, job):
    """a receive buffer shorter than the layout of the message is refused
    with BufferTooSmall for every method -- DIRECT included, whose sender
    writes the receive buffer straight from its kernel -- and no byte past
    the buffer is written"""
    import torch
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.rt as rt
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=4 << 20, host_bytes=4 << 20)
    ct = sp.commit_type(sp.make_vector(256, 4, 8, sp.make_named(sp.NamedKind.Double)))  # 8 KiB at 16 KiB span
    seen = []
    for i, method in enumerate((rt.DIRECT, rt.DEVICE, rt.ONESHOT, rt.STAGED, rt.AUTO)):
        if rank == 0:
            src = torch.arange(ct.span, dtype=torch.uint8, device="cuda")
            try:
                rt.send(src, 1, ct, 1, tag=i, method=method)
            except sp.Error:
                pass
        else:
            full = torch.full((ct.span + 4096,), 0x5A, dtype=torch.uint8, device="cuda")
            try:
                rt.recv(full[:ct.span - 8], 1, ct, source=0, tag=i)
                seen.append("accepted")
            except sp.BufferTooSmall:
                seen.append("refused")
            torch.cuda.synchronize()
            tail = full[ct.span - 8:].cpu()
            assert bool((tail == 0x5A).all()), (method, "bytes written past the receive buffer")
        rt.barrier()
    rt.finalize()
    return seen


@pytest.mark.gpu
def test_recv_buffer_too_small_every_method(cuda):
    res = _spawn(_recv_buffer_too_small, 2)
    assert res[1] == ["refused"] * 5


def _nonblocking(rank, world, job):
    """rank 0 posts every message before rank 1 posts a single receive
    (receives posted in reverse tag order): forced methods, DIRECT, chunked
    pipelining with a 64 KiB chunk, multi-object counts, a pageable host
    source, a zero-byte message, and a truncated receive"""
    import torch
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.rt as rt
    from oracle.pyoracle import oracle
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=16 << 20, host_bytes=16 << 20)
    rt.set_chunk(64 << 10)
    progs = [[4, 3, 0, 128, 64, 16, 64, 32, 8, 16, 8, 4, 0, 0],        # 3D subarray, 16 KiB
             [4, 3, 0, 512, 96, 40, 96, 80, 36, 3, 5, 2, 0, 0],        # 276 KiB, odd start
             [2, 4096, 1, 9, 0, 3],                                   # 32 KiB vector of doubles
             [3, 700, 3, 1000, 0, 0]]                                 # hvector of 3-byte blocks
    plan = [(0, rt.DEVICE, 1), (1, rt.DEVICE, 2), (1, rt.STAGED, 1), (1, rt.ONESHOT, 2), (1, rt.DIRECT, 1),
            (0, rt.DIRECT, 3), (2, rt.AUTO, 2), (3, rt.STAGED, 4), (3, rt.DIRECT, 2), (2, rt.ONESHOT, 1)]
    types = [sp.commit_type(sp.from_program(p)) for p in progs]
    orc = oracle()
    used = []
    if rank == 0:
        reqs = []
        for tag, (ti, method, count) in enumerate(plan):
            ct = types[ti]
            span = (count - 1) * ct.extent + ct.span
            host = np.random.default_rng(tag).integers(0, 256, span, dtype=np.uint8)
            src = torch.from_numpy(host) if tag == 9 else torch.from_numpy(host).cuda()  # tag 9: pageable
            reqs.append(rt.isend(src, count, ct, 1, tag=tag, method=method))
        zero = rt.isend(torch.zeros(16, dtype=torch.uint8, device="cuda"), 0, types[0], 1, tag=50)
        trunc = rt.isend(torch.zeros(types[2].span * 2, dtype=torch.uint8, device="cuda"), 2, types[2], 1, tag=60)
        used = [r["method"] for r in rt.waitall(reqs)]
        zero.wait()
        trunc.wait()
    else:
        reqs = {}
        bufs = {}
        for tag in reversed(range(len(plan))):
            ti, method, count = plan[tag]
            ct = types[ti]
            span = (count - 1) * ct.extent + ct.span
            bufs[tag] = torch.full((span,), 0x77, dtype=torch.uint8, device="cuda")
            reqs[tag] = rt.irecv(bufs[tag], count, ct, source=0, tag=tag)
        for tag in range(len(plan)):
            ti, method, count = plan[tag]
            st = reqs[tag].wait()
            ct = types[ti]
            span = (count - 1) * ct.extent + ct.span
            host = np.random.default_rng(tag).integers(0, 256, span, dtype=np.uint8)
            packed = np.zeros(count * ct.size, np.uint8)
            assert orc.pack(progs[ti], host, count, packed, 0)[0] == 0
            want = np.full(span, 0x77, np.uint8)
            assert orc.unpack(progs[ti], packed, 0, count, want)[0] == 0
            assert np.array_equal(bufs[tag].cpu().numpy(), want), (tag, st)
            assert st["bytes"] == count * ct.size and st["tag"] == tag
            used.append(st["method"])
        z = rt.irecv(torch.zeros(16, dtype=torch.uint8, device="cuda"), 1, types[0], source=0, tag=50)
        assert z.wait()["bytes"] == 0
        t = rt.irecv(torch.zeros(types[2].span, dtype=torch.uint8, device="cuda"), 1, types[2], source=0, tag=60)
        try:
            t.wait()
            raise AssertionError("truncation not reported")
        except sp.BufferTooSmall:
            pass
    rt.finalize()
    return used


@pytest.mark.gpu
def test_nonblocking_pipelined_and_direct(cuda):
    res = _spawn(_nonblocking, 2)
    # both sides agree on the method each message used
    assert res[0] == res[1]
    m = res[0]
    assert m[0] == 1 and m[1] == 1 and m[2] == 2 and m[3] == 0  # forced DEVICE / STAGED / ONESHOT
    assert m[4] == 3 and m[5] == 3 and m[8] == 3               # DIRECT into device buffers
    assert m[9] == 0


def _window_pressure(rank, world, job):
    """24 DEVICE and 8 STAGED messages of 256 KiB in flight at once into a
    1 MiB window / host region: grants wait for space and the receiver still
    matches in posting order"""
    import torch
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.rt as rt
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=1 << 20, host_bytes=1 << 20)
    ct = sp.commit_type(sp.make_hvector(1024, 1, 512, sp.make_contiguous(256, sp.make_named(sp.NamedKind.Byte))))
    n = 32
    ok = True
    if rank == 0:
        srcs = [torch.full((1024 * 512,), k, dtype=torch.uint8, device="cuda") for k in range(n)]
        torch.cuda.synchronize()
        reqs = [rt.isend(srcs[k], 1, ct, 1, tag=7, method=rt.DEVICE if k % 4 else rt.STAGED) for k in range(n)]
        rt.waitall(reqs)
    else:
        dsts = [torch.zeros(1024 * 512, dtype=torch.uint8, device="cuda") for _ in range(n)]
        torch.cuda.synchronize()
        reqs = [rt.irecv(dsts[k], 1, ct, source=0, tag=7) for k in range(n)]
        sts = rt.waitall(reqs)
        for k in range(n):
            v = dsts[k].view(1024, 512)[:, :256]
            ok = ok and bool((v == k).all()) and bool((dsts[k].view(1024, 512)[:, 256:] == 0).all())
            ok = ok and sts[k]["bytes"] == ct.size and sts[k]["method"] == (1 if k % 4 else 2)
    rt.finalize()
    return ok


@pytest.mark.gpu
def test_many_messages_window_pressure(cuda):
    assert all(_spawn(_window_pressure, 2).values())


def _ring(rank, world, job):
    """every rank sends to its right and receives from its left at once"""
    import torch
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.rt as rt
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=8 << 20, host_bytes=8 << 20)
    rt.set_chunk(32 << 10)
    ct = sp.commit_type(sp.from_program([4, 3, 0, 256, 64, 32, 128, 40, 20, 64, 8, 6, 0, 0]))
    right, left = (rank + 1) % world, (rank - 1) % world
    ok = True
    for it, method in enumerate([rt.DEVICE, rt.DIRECT, rt.STAGED, rt.ONESHOT, rt.AUTO]):
        src = torch.full((ct.span,), rank * 16 + it, dtype=torch.uint8, device="cuda")
        dst = torch.zeros(ct.span, dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()  # MPI semantics: buffers are ready when the call is made
        r = rt.irecv(dst, 1, ct, source=left, tag=it)
        s = rt.isend(src, 1, ct, right, tag=it, method=method)
        s.wait()
        r.wait()
        want = torch.zeros(ct.span, dtype=torch.uint8, device="cuda")
        full = torch.full((ct.span,), left * 16 + it, dtype=torch.uint8, device="cuda")
        sp.unpack(*_packed(sp, ct, full), 0, ct, 1, want)
        ok = ok and bool(torch.equal(dst, want))
        assert ok, (it, method)
    rt.finalize()
    return ok


def _packed(sp, ct, full):
    import torch
    p = torch.empty(ct.size, dtype=torch.uint8, device="cuda")
    sp.pack(full, ct, 1, p, 0)
    torch.cuda.synchronize()
    return (p,)


@pytest.mark.gpu
def test_nonblocking_ring_three_processes(cuda):
    assert all(_spawn(_ring, 3).values())


def _nbrw(rank, world, job):
    """MPI_Neighbor_alltoallw on a ring of 3: repeated calls (the cached fast
    path), then the receiver switches buffers and types between calls -- the
    senders must see the new layouts (layout versions) and stay exact"""
    import torch
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.rt as rt
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=1 << 20, host_bytes=1 << 20)
    right, left = (rank + 1) % world, (rank - 1) % world
    B = sp.make_named(sp.NamedKind.Byte)
    # a 3-D 64x32x16 block of bytes; send the interior box, receive into two layouts
    box = sp.commit_type(sp.make_subarray(3, [64, 32, 16], [16, 8, 4], [8, 4, 2], B))
    dst_a = sp.commit_type(sp.make_subarray(3, [64, 32, 16], [16, 8, 4], [40, 20, 10], B))
    dst_b = sp.commit_type(sp.make_hvector(32, 1, 96, sp.make_contiguous(16, B)))  # 512 B, other shape
    n = 64 * 32 * 16
    src = torch.arange(n, dtype=torch.int64, device="cuda").mul_(7).add_(rank).to(torch.uint8)
    ok = True
    for it in range(4):
        rdt = dst_a if it < 2 else dst_b
        recv = torch.full((n + (4096 if it == 3 else 0),), 0xAB, dtype=torch.uint8, device="cuda")  # new buffer
        torch.cuda.synchronize()
        rt.NeighborW([(right, 1, box, 0)], [(left, 1, rdt, 0)])(src, recv)
        # expected: the left neighbour's box bytes, unpacked with rdt
        lsrc = torch.arange(n, dtype=torch.int64, device="cuda").mul_(7).add_(left).to(torch.uint8)
        packed = torch.empty(box.size, dtype=torch.uint8, device="cuda")
        sp.pack(lsrc, box, 1, packed, 0)
        want = torch.full_like(recv, 0xAB)
        sp.unpack(packed, 0, rdt, 1, want)
        torch.cuda.synchronize()
        ok = ok and bool(torch.equal(recv, want))
        assert ok, (rank, it)

    def expect(shift):
        lsrc = torch.arange(n, dtype=torch.int64, device="cuda").mul_(7).add_(left + shift).to(torch.uint8)
        packed = torch.empty(box.size, dtype=torch.uint8, device="cuda")
        sp.pack(lsrc, box, 1, packed, 0)
        want = torch.full_like(recv, 0xAB)
        sp.unpack(packed, 0, dst_a, 1, want)
        return want

    # identical arguments call after call (the repeat path skips the layout
    # publication and the launch lookup) while the source bytes change: every
    # call must move the current bytes
    recv = torch.full((n,), 0xAB, dtype=torch.uint8, device="cuda")
    call = rt.NeighborW([(right, 1, box, 0)], [(left, 1, dst_a, 0)])
    for shift in range(1, 4):
        src = torch.arange(n, dtype=torch.int64, device="cuda").mul_(7).add_(rank + shift).to(torch.uint8)
        torch.cuda.synchronize()
        call(src, recv)
        torch.cuda.synchronize()
        assert torch.equal(recv, expect(shift)), (rank, "repeat", shift)
    rt.finalize()
    # a new runtime in the same process: the same call must not reuse the
    # previous runtime's launches (they name its IPC mappings)
    rt.init(rank, world, job + "b", device=0, window_bytes=1 << 20, host_bytes=1 << 20)
    recv.fill_(0xAB)
    src = torch.arange(n, dtype=torch.int64, device="cuda").mul_(7).add_(rank + 9).to(torch.uint8)
    torch.cuda.synchronize()
    call(src, recv)
    torch.cuda.synchronize()
    assert torch.equal(recv, expect(9)), (rank, "re-init")
    # a handle freed between calls: the memoised handle lookups must notice
    # (MPI_ERR_TYPE territory), not reuse the freed type's record
    from paper_2012_14363_b200 import _capi
    import ctypes as C
    extra = sp.make_contiguous(16, B)
    assert _capi.lib.sp_type_commit(extra.handle) == 0
    hs = (_capi.sp_type * 1)(extra.handle)
    sc = (C.c_int64 * 1)(0)
    nb = (C.c_int * 1)(rank)
    lib = _capi.lib
    assert lib.sp_rt_neighbor_alltoallw(src.data_ptr(), sc, sc, hs, 1, nb, recv.data_ptr(), sc, sc, hs, 1, nb) == 0
    assert lib.sp_type_free(extra.handle) == 0
    st = lib.sp_rt_neighbor_alltoallw(src.data_ptr(), sc, sc, hs, 1, nb, recv.data_ptr(), sc, sc, hs, 1, nb)
    assert st == 11, st  # SP_ERR_INVALID_HANDLE
    extra.handle = 0  # already freed
    rt.finalize()
    return ok


@pytest.mark.gpu
def test_neighbor_alltoallw_layout_changes(cuda):
    assert all(_spawn(_nbrw, 3).values())


def _nbrv(rank, world, job):
    """MPI_Neighbor_alltoallv on a ring of 3 with a packed (bytes) and a
    strided receive type, 2 objects per edge, displacements in extents"""
    import torch
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.rt as rt
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=1 << 20, host_bytes=1 << 20)
    right, left = (rank + 1) % world, (rank - 1) % world
    B = sp.make_named(sp.NamedKind.Byte)
    st = sp.commit_type(sp.make_vector(8, 24, 64, B))               # 192 B per object, extent 472
    dense = sp.commit_type(sp.make_contiguous(192, B))
    strided = sp.commit_type(sp.make_hvector(12, 16, 40, B))        # 192 B, extent 456
    src = torch.arange(4096, dtype=torch.int64, device="cuda").mul_(13).add_(rank * 7).to(torch.uint8)
    lsrc = torch.arange(4096, dtype=torch.int64, device="cuda").mul_(13).add_(left * 7).to(torch.uint8)
    rsrc = torch.arange(4096, dtype=torch.int64, device="cuda").mul_(13).add_(right * 7).to(torch.uint8)
    ok = True
    for rt_type in (dense, strided):
        for it in range(2):
            recv = torch.full((8192,), 0xEE, dtype=torch.uint8, device="cuda")
            torch.cuda.synchronize()
            # 2 objects to the right at displacement 1, 2 objects to the left at displacement 4
            rt.neighbor_alltoallv(src, st, [(right, 2, 1), (left, 2, 4)], recv, rt_type, [(left, 2, 0), (right, 2, 6)])
            want = torch.full_like(recv, 0xEE)
            pk = torch.empty(2 * 192, dtype=torch.uint8, device="cuda")
            for peer_src, sdisp, rdisp in ((lsrc, 1, 0), (rsrc, 4, 6)):
                sp.pack(peer_src[sdisp * st.extent:], st, 2, pk, 0)
                sp.unpack(pk, 0, rt_type, 2, want[rdisp * rt_type.extent:])
            torch.cuda.synchronize()
            ok = ok and bool(torch.equal(recv, want))
            assert ok, (rank, rt_type is strided, it)
    rt.finalize()
    return ok


@pytest.mark.gpu
def test_neighbor_alltoallv_packed_and_strided_receive(cuda):
    assert all(_spawn(_nbrv, 3).values())


def _nbr_irregular(rank, world, job):
    """Unstructured-mesh style neighbour exchange: each rank sends an
    irregular MPI_Type_indexed gather list (different per neighbour, so not
    one strided form) and receives contiguous ghost runs.
    MPI_Neighbor_alltoallw (per-edge types) and MPI_Neighbor_alltoallv (one
    irregular send type, packed receive), repeated (the cached fast path)
    with changing source data, on a ring of 3."""
    import numpy as np
    import torch
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.rt as rt
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=1 << 20, host_bytes=1 << 20)
    right, left = (rank + 1) % world, (rank - 1) % world
    D = sp.make_named(sp.NamedKind.Double)

    def gather_list(seed):
        g = np.random.default_rng(seed)
        n = 300
        bl = g.integers(1, 4, n).tolist()
        slots = g.permutation(1024)[:n]
        return bl, [int(x) * 4 for x in slots]  # blocks of <= 3 doubles in 4-double slots

    def itype(seed):
        bl, dp = gather_list(seed)
        return sp.commit_type(sp.make_indexed(bl, dp, D)), bl, dp

    # edge types keyed by (sender, receiver): both ends build the same list
    t_r, bl_r, dp_r = itype(100 * rank + right)
    t_l, bl_l, dp_l = itype(100 * rank + left)
    _, bl_in_l, dp_in_l = itype(100 * left + rank)    # what the left neighbour sends me
    _, bl_in_r, dp_in_r = itype(100 * right + rank)
    n_from_l, n_from_r = sum(bl_in_l), sum(bl_in_r)
    ghost_l = sp.commit_type(sp.make_contiguous(n_from_l, D))
    ghost_r = sp.commit_type(sp.make_contiguous(n_from_r, D))
    N = 4096
    field = torch.empty(N, dtype=torch.float64, device="cuda")
    recv = torch.empty(n_from_l + n_from_r + 8, dtype=torch.float64, device="cuda")

    def values(r, it):
        return torch.arange(N, dtype=torch.float64, device="cuda") * 3 + r * 100000 + it

    def expect_from(r, bl, dp, it):
        v = values(r, it).cpu().numpy()
        return np.concatenate([v[d:d + b] for b, d in zip(bl, dp)])

    call = rt.NeighborW([(right, 1, t_r, 0), (left, 1, t_l, 0)],
                        [(left, 1, ghost_l, 0), (right, 1, ghost_r, 8 * n_from_l)])
    for it in range(4):
        field.copy_(values(rank, it))
        recv.fill_(-1)
        torch.cuda.synchronize()
        call(field, recv)
        torch.cuda.synchronize()
        got = recv.cpu().numpy()
        assert np.array_equal(got[:n_from_l], expect_from(left, bl_in_l, dp_in_l, it)), (rank, it, "left")
        assert np.array_equal(got[n_from_l:n_from_l + n_from_r], expect_from(right, bl_in_r, dp_in_r, it)), (rank, it)
        assert (got[n_from_l + n_from_r:] == -1).all()
    # alltoallv: one irregular send type for both neighbours, packed receive
    tv, blv, dpv = itype(7)  # the same list on every rank
    nv = sum(blv)
    packed = sp.commit_type(sp.make_contiguous(8, sp.make_named(sp.NamedKind.Byte)))  # one double
    for it in range(3):
        field.copy_(values(rank, 10 + it))
        recv2 = torch.full((2 * nv,), -1.0, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        rt.neighbor_alltoallv(field, tv, [(right, 1, 0), (left, 1, 0)], recv2, packed,
                              [(left, nv, 0), (right, nv, nv)])
        torch.cuda.synchronize()
        got = recv2.cpu().numpy()
        assert np.array_equal(got[:nv], expect_from(left, blv, dpv, 10 + it)), (rank, it, "v-left")
        assert np.array_equal(got[nv:], expect_from(right, blv, dpv, 10 + it)), (rank, it, "v-right")
    # the alltoallw again with identical arguments: the alltoallv in between
    # published another receive layout, so the repeat path must not skip
    # re-publishing this call's layout
    field.copy_(values(rank, 20))
    recv.fill_(-1)
    torch.cuda.synchronize()
    call(field, recv)
    torch.cuda.synchronize()
    got = recv.cpu().numpy()
    assert np.array_equal(got[:n_from_l], expect_from(left, bl_in_l, dp_in_l, 20)), (rank, "w-again")
    assert np.array_equal(got[n_from_l:n_from_l + n_from_r], expect_from(right, bl_in_r, dp_in_r, 20))
    rt.finalize()
    return True


def _nbr_irregular_recv(rank, world, job):
    """Scattered ghosts: each rank sends a contiguous run of doubles to each
    neighbour and receives it through an irregular MPI_Type_indexed
    (different per neighbour) -- the sender scatters through the receiver's
    run table published over CUDA IPC. Repeated calls with changing data,
    ring of 3."""
    import numpy as np
    import torch
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.rt as rt
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=1 << 20, host_bytes=1 << 20)
    right, left = (rank + 1) % world, (rank - 1) % world
    D = sp.make_named(sp.NamedKind.Double)

    def scatter_list(seed, lo):
        g = np.random.default_rng(seed)
        bl = g.integers(1, 4, 200).tolist()
        slots = g.permutation(512)[:200]
        return bl, [lo + int(x) * 4 for x in slots]

    # my ghost layout for data from the left lives in [0, 2048) doubles, from the right in [2048, 4096)
    bl_l, dp_l = scatter_list(100 * rank + left, 0)
    bl_r, dp_r = scatter_list(100 * rank + right, 2048)
    g_l = sp.commit_type(sp.make_indexed(bl_l, dp_l, D))
    g_r = sp.commit_type(sp.make_indexed(bl_r, dp_r, D))
    # what my neighbours expect from me: the sizes of THEIR lists for me
    n_to_r = sum(scatter_list(100 * right + rank, 0)[0])
    n_to_l = sum(scatter_list(100 * left + rank, 2048)[0])
    s_r = sp.commit_type(sp.make_contiguous(n_to_r, D))
    s_l = sp.commit_type(sp.make_contiguous(n_to_l, D))
    src = torch.empty(n_to_r + n_to_l, dtype=torch.float64, device="cuda")
    ghosts = torch.empty(4096, dtype=torch.float64, device="cuda")
    call = rt.NeighborW([(right, 1, s_r, 0), (left, 1, s_l, 8 * n_to_r)],
                        [(left, 1, g_l, 0), (right, 1, g_r, 0)])

    def sent_by(r, to_right, it):
        # rank r sends [0, n) to its right neighbour and [n, n + m) to its left
        n = sum(scatter_list(100 * ((r + 1) % world) + r, 0)[0])
        m = sum(scatter_list(100 * ((r - 1) % world) + r, 2048)[0])
        v = np.arange(n + m, dtype=np.float64) * 7 + r * 1000 + it
        return v[:n] if to_right else v[n:]

    for it in range(3):
        src.copy_(torch.from_numpy(np.arange(n_to_r + n_to_l, dtype=np.float64) * 7 + rank * 1000 + it))
        ghosts.fill_(-1)
        torch.cuda.synchronize()
        call(src, ghosts)
        torch.cuda.synchronize()
        want = np.full(4096, -1.0)
        for bl, dp, vals in ((bl_l, dp_l, sent_by(left, True, it)), (bl_r, dp_r, sent_by(right, False, it))):
            k = 0
            for b, d in zip(bl, dp):
                want[d:d + b] = vals[k:k + b]
                k += b
        assert np.array_equal(ghosts.cpu().numpy(), want), (rank, it)
    rt.finalize()
    return True


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_neighbor_alltoallw_irregular_receive_types(cuda, world):
    assert all(_spawn(_nbr_irregular_recv, world).values())


def _nbr_misaligned_runs(rank, world, job):
    """Byte-granular irregular edges (hindexed of MPI_BYTE, odd lengths and
    displacements, mean run ~1 KiB): the shift variant of the run-table
    kernel (k_runs_multi_shift) for gathers into contiguous ghosts (first
    call) and for scatters of contiguous runs through the receivers'
    published run tables (second call); ring, verified byte by byte."""
    import numpy as np
    import torch
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.rt as rt
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=1 << 20, host_bytes=1 << 20)
    right, left = (rank + 1) % world, (rank - 1) % world
    B = sp.make_named(sp.NamedKind.Byte)

    def runs(seed, lo):  # 35 runs of 600-1400 B at odd, non-overlapping offsets inside [lo, lo + 65536)
        g = np.random.default_rng(seed)
        bl = g.integers(600, 1401, 35)
        at = lo + 3 + np.concatenate([[0], np.cumsum(bl + g.integers(1, 300, 35))[:-1]])
        perm = g.permutation(35)
        return [int(x) for x in bl[perm]], [int(x) for x in at[perm]]

    def expect(bl, dp, vals, base, n):
        want = np.full(n, 0xEE, np.uint8)
        k = 0
        for b, d in zip(bl, dp):
            want[d - base:d - base + b] = vals[k:k + b]
            k += b
        return want

    field = torch.from_numpy((np.arange(1 << 17) * 7 + rank * 31).astype(np.uint8)).cuda()
    host_field = lambda r: (np.arange(1 << 17) * 7 + r * 31).astype(np.uint8)
    # 1. gathers: my irregular lists for each neighbour -> their contiguous ghosts
    bl_r, dp_r = runs(10 * rank + right, 0)
    bl_l, dp_l = runs(10 * rank + left, 65536)
    in_l, in_r = runs(10 * left + rank, 0), runs(10 * right + rank, 65536)
    n_l, n_r = sum(in_l[0]), sum(in_r[0])
    call = rt.NeighborW([(right, 1, sp.commit_type(sp.make_hindexed(bl_r, dp_r, B)), 0),
                         (left, 1, sp.commit_type(sp.make_hindexed(bl_l, dp_l, B)), 0)],
                        [(left, 1, sp.commit_type(sp.make_contiguous(n_l, B)), 0),
                         (right, 1, sp.commit_type(sp.make_contiguous(n_r, B)), n_l)])
    ghosts = torch.full((n_l + n_r,), 0xEE, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    call(field, ghosts)
    torch.cuda.synchronize()
    got = ghosts.cpu().numpy()
    want_l = np.concatenate([host_field(left)[d:d + b] for b, d in zip(*in_l)])
    want_r = np.concatenate([host_field(right)[d:d + b] for b, d in zip(*in_r)])
    assert np.array_equal(got[:n_l], want_l) and np.array_equal(got[n_l:], want_r), rank
    # 2. scatters: contiguous runs -> my irregular ghost layouts
    g_l, g_r = runs(20 * rank + left, 0), runs(20 * rank + right, 65536)
    out_r, out_l = runs(20 * right + rank, 0), runs(20 * left + rank, 65536)  # my neighbours' layouts for me
    m_r, m_l = sum(out_r[0]), sum(out_l[0])
    call2 = rt.NeighborW([(right, 1, sp.commit_type(sp.make_contiguous(m_r, B)), 0),
                          (left, 1, sp.commit_type(sp.make_contiguous(m_l, B)), m_r)],
                         [(left, 1, sp.commit_type(sp.make_hindexed(*g_l, B)), 0),
                          (right, 1, sp.commit_type(sp.make_hindexed(*g_r, B)), 0)])
    src = torch.from_numpy((np.arange(m_r + m_l) * 5 + rank).astype(np.uint8)).cuda()
    recv = torch.full((1 << 17,), 0xEE, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    call2(src, recv)
    torch.cuda.synchronize()
    sent = lambda r, n, off: (np.arange(off, off + n) * 5 + r).astype(np.uint8)
    # the left neighbour's block for its right (me) is its first; the right
    # neighbour's block for its left (me) follows its block for ITS right
    vals_l = sent(left, sum(g_l[0]), 0)
    vals_r = sent(right, sum(g_r[0]), sum(runs(20 * ((right + 1) % world) + right, 0)[0]))
    want = expect(*g_l, vals_l, 0, 1 << 17)
    k = 0
    for b, d in zip(*g_r):
        want[d:d + b] = vals_r[k:k + b]
        k += b
    assert np.array_equal(recv.cpu().numpy(), want), rank
    rt.finalize()
    return True


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_neighbor_misaligned_irregular_runs(cuda, world):
    assert all(_spawn(_nbr_misaligned_runs, world).values())


def _nbr_alternating_layouts(rank, world, job, iters):
    """Regression for the shared neighbour protocol (entry counters, READY
    flags, layout versions, repeat-call and batch caches): every rank of a
    ring alternates its receive layout between four REGULAR types on
    every call, verified cell by cell each time. Layouts C and D have the
    same canonical geometry (one dense 32-B row) and differ only in extent,
    so a batch cached under a key without the receiver's extent would put
    object j at the wrong pitch."""
    import numpy as np
    import torch
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.rt as rt
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=1 << 20, host_bytes=1 << 20)
    right, left = (rank + 1) % world, (rank - 1) % world
    D = sp.make_named(sp.NamedKind.Double)
    flat = sp.commit_type(sp.make_contiguous(128, D))
    idx = lambda blocks: np.concatenate([np.arange(o, o + n) for o, n in blocks])
    layouts = [  # (type, count, element indices of the 128 received doubles)
        (sp.commit_type(sp.make_vector(64, 2, 5, D)), 1, idx([(5 * b, 2) for b in range(64)])),
        (sp.commit_type(sp.make_vector(32, 4, 7, D)), 1, idx([(7 * b, 4) for b in range(32)])),
        (sp.commit_type(sp.make_contiguous(4, D)), 32, np.arange(128)),
        (sp.commit_type(sp.make_subarray(1, [8], [4], [0], D)), 32, idx([(8 * j, 4) for j in range(32)])),
    ]
    assert layouts[2][0].canon.counts == layouts[3][0].canon.counts and layouts[2][0].extent != layouts[3][0].extent
    calls = [rt.NeighborW([(right, 1, flat, 0), (left, 1, flat, 8 * 128)],
                          [(left, c, t, 0), (right, c, t, 8 * 1024)]) for t, c, _ in layouts]
    send = torch.empty(256, dtype=torch.float64, device="cuda")
    recv = torch.empty(2048, dtype=torch.float64, device="cuda")
    sent = lambda r, it: np.arange(256, dtype=np.float64) + r * 1e6 + it * 1e3
    bad, detail = 0, []
    for it in range(iters):
        k = (it + rank) % len(layouts) if it % 3 else it % len(layouts)  # ranks disagree on most calls
        send.copy_(torch.from_numpy(sent(rank, it)))
        recv.fill_(-1)
        torch.cuda.synchronize()  # the buffers are ready before the call (MPI's rule for device buffers)
        calls[k](send, recv)
        want = np.full(2048, -1.0)
        want[layouts[k][2]] = sent(left, it)[:128]           # left sent me its first run
        want[1024 + layouts[k][2]] = sent(right, it)[128:]   # right sent me its second run
        got = recv.cpu().numpy()
        if not np.array_equal(got, want):
            bad += 1
            if len(detail) < 4:
                wrong = np.nonzero(got != want)[0]
                detail.append((it, k, len(wrong), int(wrong[0]), float(got[wrong[0]]), float(want[wrong[0]])))
    rt.finalize()
    return bad, detail


@pytest.mark.gpu
def test_neighbor_alltoallw_alternating_layouts(cuda):
    res = _spawn(_nbr_alternating_layouts, 3, 1000, timeout=600)
    assert all(bad == 0 for bad, _ in res.values()), res


def _nbr_error_after_entry(rank, world, job):
    """one rank's send disagrees with its neighbour's receive (refused only
    after the call was entered): that rank gets the error, the other rank's
    call still completes instead of hanging its GPU, and the next correct
    call on the same pair is exact (the per-pair call counts stay in step)"""
    import numpy as np
    import torch
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.rt as rt
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=1 << 20, host_bytes=1 << 20)
    peer = 1 - rank
    D = sp.make_named(sp.NamedKind.Double)
    t128, t64 = sp.commit_type(sp.make_contiguous(128, D)), sp.commit_type(sp.make_contiguous(64, D))
    send = torch.arange(128, dtype=torch.float64, device="cuda") + rank * 1000
    recv = torch.full((128,), -1.0, dtype=torch.float64, device="cuda")
    bad = rt.NeighborW([(peer, 1, t64 if rank == 1 else t128, 0)], [(peer, 1, t128, 0)])
    err = None
    try:
        bad(send, recv)
    except sp.Error as e:
        err = type(e).__name__
    good = rt.NeighborW([(peer, 1, t128, 0)], [(peer, 1, t128, 0)])
    recv.fill_(-1)
    good(send, recv)
    torch.cuda.synchronize()
    exact = bool(np.array_equal(recv.cpu().numpy(), np.arange(128) + peer * 1000.0))
    rt.finalize()
    return err, exact


@pytest.mark.gpu
def test_neighbor_error_after_entry_does_not_hang_peers(cuda):
    res = _spawn(_nbr_error_after_entry, 2, timeout=120)
    assert res[1] == ("InvalidArgument", True) and res[0][1] is True, res


def _nbr_many_irregular(rank, world, job):
    """40 irregular edges to self in one MPI_Neighbor_alltoallw: more than
    one run-table launch's worth of edges (32 per launch)"""
    import numpy as np
    import torch
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.rt as rt
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=1 << 20, host_bytes=1 << 20)
    D = sp.make_named(sp.NamedKind.Double)
    g = np.random.default_rng(4)
    field = torch.randn(1 << 16, dtype=torch.float64, device="cuda")
    sends, recvs, lists, at = [], [], [], 0
    for e in range(40):
        bl = g.integers(1, 4, 50).tolist()
        dp = [int(x) * 4 for x in g.choice(1 << 14, 50, replace=False)]
        t = sp.commit_type(sp.make_indexed(bl, dp, D))
        n = sum(bl)
        sends.append((rank, 1, t, 0))
        recvs.append((rank, 1, sp.commit_type(sp.make_contiguous(n, D)), at * 8))
        lists.append((bl, dp, at))
        at += n
    recv = torch.zeros(at, dtype=torch.float64, device="cuda")
    before = sp.kernel_launch_count()
    rt.NeighborW(sends, recvs)(field, recv)
    torch.cuda.synchronize()
    assert sp.kernel_launch_count() - before == 2  # 32 + 8 edges
    f = field.cpu().numpy()
    r = recv.cpu().numpy()
    for bl, dp, off in lists:
        want = np.concatenate([f[d:d + b] for b, d in zip(bl, dp)])
        assert np.array_equal(r[off:off + len(want)], want)
    rt.finalize()
    return True


@pytest.mark.gpu
def test_neighbor_alltoallw_many_irregular_edges(cuda):
    assert all(_spawn(_nbr_many_irregular, 1).values())


@pytest.mark.gpu
def test_neighbor_collectives_with_irregular_send_types(cuda):
    assert all(_spawn(_nbr_irregular, 3).values())


def _halo_soak(rank, world, job, ranks, method, iters):
    """many back-to-back iterations with no barrier between them (the
    in-kernel flags alone order the ranks against each other), three rounds
    of fresh plans on reset ghosts, every cell verified after each round"""
    import torch
    import paper_2012_14363_b200.halo as H
    import paper_2012_14363_b200.rt as rt
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=1 << 20, host_bytes=1 << 20)
    cfg = H.HaloConfig(ranks, (10, 12, 8), 2, 8)
    alloc = torch.empty(14 * 16 * 12 * 8, dtype=torch.uint8, device="cuda")
    bad = 0
    for rnd in range(3):
        H.fill(cfg, rank, alloc)
        torch.cuda.synchronize()
        rt.barrier()
        plan = rt.HaloPlan(cfg, alloc, method)
        for i in range(iters):
            plan.exchange(timed=(rnd == 0))  # rounds 1-2: enqueue only, no host sync at all
        torch.cuda.ExternalStream(rt.stream()).synchronize()
        bad += H.verify(cfg, rank, alloc)
        plan.free()
    rt.finalize()
    return bad


@pytest.mark.gpu
@pytest.mark.parametrize("ranks,method", [((2, 1, 1), 3), ((1, 3, 1), 3), ((2, 1, 1), 2), ((2, 2, 1), 3)])
def test_distributed_halo_soak(cuda, ranks, method):
    world = ranks[0] * ranks[1] * ranks[2]
    res = _spawn(_halo_soak, world, ranks, method, 25, timeout=400)
    assert all(v == 0 for v in res.values()), res


def _halo(rank, world, job, ranks, method):
    import torch
    import paper_2012_14363_b200.halo as H
    import paper_2012_14363_b200.rt as rt
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=1 << 20, host_bytes=1 << 20)
    cfg = H.HaloConfig(ranks, (12, 10, 8), 2, 16)
    pad = 16 * 14 * 12 * 16
    alloc = torch.empty(pad, dtype=torch.uint8, device="cuda")
    H.fill(cfg, rank, alloc)
    plan = rt.HaloPlan(cfg, alloc, method)
    for _ in range(3):
        t = plan.exchange()
    bad = H.verify(cfg, rank, alloc)
    # reset the ghosts: a fourth iteration must rewrite all of them
    H.fill(cfg, rank, alloc)
    torch.cuda.synchronize()
    rt.barrier()
    plan.exchange()
    bad += H.verify(cfg, rank, alloc)
    plan.free()
    rt.finalize()
    return bad, t


def _halo_graph(rank, world, job, ranks, method, flag_wait):
    """a distributed exchange captured into a CUDA graph: the plan numbers
    its iterations on the device (a tick kernel advances its counter, the
    copy kernels -- or, with ranks sharing a GPU, a one-warp wait kernel
    ahead of them -- derive FREE/READY from it), so replays order the ranks
    like eager calls; host-numbered iterations before the capture and eager
    ones after it continue the same count."""
    import os
    os.environ["TEMPI_FLAG_WAIT"] = flag_wait
    import torch
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.halo as H
    import paper_2012_14363_b200.rt as rt
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=1 << 20, host_bytes=1 << 20)
    cfg = H.HaloConfig(ranks, (10, 12, 8), 2, 8)
    alloc = torch.empty(14 * 16 * 12 * 8, dtype=torch.uint8, device="cuda")
    plan = rt.HaloPlan(cfg, alloc, method)
    rs = torch.cuda.ExternalStream(rt.stream())
    H.fill(cfg, rank, alloc)
    torch.cuda.synchronize()
    rt.barrier()
    for _ in range(2):  # host-numbered iterations first
        plan.exchange(timed=False)
    rs.synchronize()
    bad = H.verify(cfg, rank, alloc)
    g = torch.cuda.CUDAGraph()
    refused = False
    with torch.cuda.stream(rs):
        g.capture_begin()
        try:
            plan.exchange(timed=False)
        except sp.Unsupported:
            refused = True
        finally:
            g.capture_end()
    if refused:
        plan.exchange()  # still usable eagerly
        bad += H.verify(cfg, rank, alloc)
        plan.free()
        rt.finalize()
        return bad, "refused"
    for _ in range(4):
        H.fill(cfg, rank, alloc)  # reset the ghosts: each replay must rewrite them
        torch.cuda.synchronize()
        rt.barrier()
        with torch.cuda.stream(rs):
            g.replay()
        rs.synchronize()
        bad += H.verify(cfg, rank, alloc)
    for _ in range(3):  # several replays back to back, no host sync between them
        with torch.cuda.stream(rs):
            g.replay()
    rs.synchronize()
    H.fill(cfg, rank, alloc)
    torch.cuda.synchronize()
    rt.barrier()
    plan.exchange(timed=False)  # eager again: device-numbered from now on
    rs.synchronize()
    bad += H.verify(cfg, rank, alloc)
    del g
    plan.free()
    rt.finalize()
    return bad, "captured"


@pytest.mark.gpu
@pytest.mark.parametrize("ranks,method", [((2, 1, 1), 3), ((2, 1, 1), 2), ((2, 2, 1), 3)])
def test_distributed_halo_graph_capture(cuda, ranks, method):
    world = ranks[0] * ranks[1] * ranks[2]
    res = _spawn(_halo_graph, world, ranks, method, "kernel", timeout=400)
    assert all(v == (0, "captured") for v in res.values()), res


@pytest.mark.gpu
@pytest.mark.parametrize("method", [3, 2])
def test_distributed_halo_graph_capture_stream_mode(cuda, method):
    """ranks sharing a GPU (stream flag waits, the default here)"""
    res = _spawn(_halo_graph, 2, (2, 1, 1), method, "stream", timeout=300)
    assert all(v == (0, "captured") for v in res.values()), res


def _nbr_plan_graph(rank, world, job, ranks, flag_wait):
    """MPI-4 persistent neighbour alltoallw (rt.NeighborPlan): the halo's 26
    region types compiled once, started eagerly, then captured into a CUDA
    graph and replayed; every ghost verified after each round"""
    import os
    os.environ["TEMPI_FLAG_WAIT"] = flag_wait
    import torch
    import paper_2012_14363_b200.halo as H
    import paper_2012_14363_b200.rt as rt
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=1 << 20, host_bytes=1 << 20)
    cfg = H.HaloConfig(ranks, (10, 12, 8), 2, 8)
    regions = H.build_halo_types(cfg)
    alloc = torch.empty(14 * 16 * 12 * 8, dtype=torch.uint8, device="cuda")
    sends = [(H.neighbor(cfg, rank, r.dir), 1, r.send, 0) for r in regions]
    recvs = [(H.neighbor(cfg, rank, tuple(-x for x in r.dir)), 1, regions[25 - j].recv, 0)
             for j, r in enumerate(regions)]
    plan = rt.NeighborPlan(sends, recvs, alloc, alloc)
    rs = torch.cuda.ExternalStream(rt.stream())
    bad = 0
    for _ in range(3):  # eager starts
        H.fill(cfg, rank, alloc)
        torch.cuda.synchronize()
        rt.barrier()
        plan.start()
        plan.wait()
        bad += H.verify(cfg, rank, alloc)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(rs):
        g.capture_begin()
        plan.start()
        g.capture_end()
    for _ in range(3):  # replays
        H.fill(cfg, rank, alloc)
        torch.cuda.synchronize()
        rt.barrier()
        with torch.cuda.stream(rs):
            g.replay()
        rs.synchronize()
        bad += H.verify(cfg, rank, alloc)
    del g
    plan.free()
    rt.finalize()
    return bad


@pytest.mark.gpu
@pytest.mark.parametrize("ranks,flag_wait", [((1, 1, 1), "stream"), ((2, 1, 1), "stream"), ((2, 2, 1), "stream"),
                                             ((2, 1, 1), "kernel")])
def test_persistent_neighbor_plan_eager_and_graph(cuda, ranks, flag_wait):
    world = ranks[0] * ranks[1] * ranks[2]
    res = _spawn(_nbr_plan_graph, world, ranks, flag_wait, timeout=400)
    assert all(v == 0 for v in res.values()), res


def _realloc_receivers(rank, world, job):
    """Receivers that free their buffer and allocate a new one (a real
    cudaFree + cudaMalloc: empty_cache between, so the new buffer usually
    lands at the old address with a new IPC handle). The sender's cached
    mapping of the old allocation is stale; it must be closed before the new
    handle is opened, for a DIRECT point-to-point destination (published with
    its pointer in the descriptor) and for a neighbour call's receive buffer
    (published in the rank's slot). Every round is checked element by
    element; returns (bad rounds, distinct receive addresses seen)."""
    import numpy as np
    import torch
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.rt as rt
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=1 << 20, host_bytes=1 << 20)
    peer = 1 - rank
    n = 1 << 16
    D = sp.make_named(sp.NamedKind.Double)
    dense = sp.commit_type(sp.make_contiguous(n, D))
    every_other = sp.commit_type(sp.make_vector(n, 1, 2, D))
    bad, addrs = 0, set()
    for it in range(6):
        # point to point, rank 0 -> rank 1, DIRECT into a strided layout
        if rank == 0:
            src = torch.arange(n, dtype=torch.float64, device="cuda") + 1000.0 * it
            torch.cuda.synchronize()
            rt.send(src, 1, dense, 1, tag=it, method=rt.DIRECT)
            del src
        else:
            dst = torch.full((2 * n,), -1.0, dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            addrs.add(dst.data_ptr())
            st = rt.recv(dst, 1, every_other, 0, it)
            h = dst.cpu().numpy()
            bad += not (st["method"] == rt.DIRECT and np.array_equal(h[0::2], np.arange(n) + 1000.0 * it)
                        and (h[1::2] == -1).all())
            del dst
        torch.cuda.empty_cache()
        rt.barrier()
        # a neighbour alltoallw both ways into fresh receive buffers
        src = torch.arange(n, dtype=torch.float64, device="cuda") + 1e6 * rank + it
        dst = torch.full((2 * n,), -1.0, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        rt.NeighborW([(peer, 1, dense, 0)], [(peer, 1, every_other, 0)])(src, dst)
        torch.cuda.synchronize()
        h = dst.cpu().numpy()
        bad += not (np.array_equal(h[0::2], np.arange(n) + 1e6 * peer + it) and (h[1::2] == -1).all())
        del src, dst
        torch.cuda.empty_cache()
        rt.barrier()
    rt.finalize()
    return bad, len(addrs)


@pytest.mark.gpu
def test_receivers_reallocating_buffers(cuda):
    res = _spawn(_realloc_receivers, 2, timeout=300)
    assert all(v[0] == 0 for v in res.values()), res


def _nbr_plan_refused(rank, world, job):
    """only rank 0 has a receive type the plan cannot compile (an irregular
    indexed layout): every rank must refuse the plan together (a rank that
    went on alone would wait forever in the creation's barriers), and an
    ordinary call still works afterwards"""
    import numpy as np
    import torch
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.rt as rt
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=1 << 20, host_bytes=1 << 20)
    peer = 1 - rank
    D = sp.make_named(sp.NamedKind.Double)
    flat = sp.commit_type(sp.make_contiguous(6, D))
    irregular = sp.commit_type(sp.make_indexed([2, 1, 3], [9, 0, 4], D))
    recv_t = irregular if rank == 0 else flat
    src = torch.arange(6, dtype=torch.float64, device="cuda") + 100 * rank
    dst = torch.full((16,), -1.0, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    refused = False
    try:
        rt.NeighborPlan([(peer, 1, flat, 0)], [(peer, 1, recv_t, 0)], src, dst)
    except sp.Unsupported:
        refused = True
    rt.NeighborW([(peer, 1, flat, 0)], [(peer, 1, recv_t, 0)])(src, dst)
    torch.cuda.synchronize()
    got = dst.cpu().numpy()
    sent = np.arange(6) + 100 * peer
    if rank == 0:
        want = np.full(16, -1.0)
        k = 0
        for b, d in zip([2, 1, 3], [9, 0, 4]):
            want[d:d + b] = sent[k:k + b]
            k += b
    else:
        want = np.concatenate([sent, np.full(10, -1.0)])
    rt.finalize()
    return refused and bool(np.array_equal(got, want))


@pytest.mark.gpu
def test_persistent_neighbor_plan_refused_together(cuda):
    assert all(_spawn(_nbr_plan_refused, 2, timeout=200).values())


def _halo_peer_absent(rank, world, job):
    """rank 1 builds the DIRECT halo plan and then never exchanges: rank 0's
    exchange kernel waits in its last block for rank 1's READY flag, gives
    up after TEMPI_TIMEOUT, and the host reports Timeout instead of the GPU
    spinning forever"""
    import time
    import torch
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.halo as H
    import paper_2012_14363_b200.rt as rt
    torch.cuda.set_device(0)
    rt.init(rank, world, job, device=0, window_bytes=1 << 20, host_bytes=1 << 20)
    cfg = H.HaloConfig((2, 1, 1), (12, 10, 8), 2, 16)
    alloc = torch.empty(16 * 14 * 12 * 16, dtype=torch.uint8, device="cuda")
    plan = rt.HaloPlan(cfg, alloc, 3)
    if rank == 1:
        time.sleep(8)
        return "absent"
    t0 = time.time()
    try:
        plan.exchange()
        return "no error"
    except sp.Timeout:
        return ("Timeout", time.time() - t0 < 7)


@pytest.mark.gpu
def test_device_flag_wait_times_out(cuda, monkeypatch):
    monkeypatch.setenv("TEMPI_TIMEOUT", "2")
    res = _spawn_raw(_halo_peer_absent, 2, timeout=120)
    assert res.get(0) == ("Timeout", True), res


@pytest.mark.gpu
@pytest.mark.parametrize("ranks,method", [((2, 1, 1), 0), ((2, 1, 1), 1), ((1, 3, 1), 0), ((1, 1, 1), 2),
                                          ((2, 1, 1), 2), ((2, 2, 1), 2), ((1, 1, 1), 3), ((2, 1, 1), 3),
                                          ((1, 3, 1), 3), ((2, 2, 1), 3)])
def test_distributed_halo_exchange(cuda, ranks, method):
    world = ranks[0] * ranks[1] * ranks[2]
    res = _spawn(_halo, world, ranks, method)
    for r, (bad, t) in res.items():
        assert bad == 0, (r, bad)
        assert t["pack"] > 0 and t["iteration"] >= t["pack"]
