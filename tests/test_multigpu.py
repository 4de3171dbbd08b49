"""Multi-GPU validation: one process per DISTINCT device, so every IPC
mapping, system-scope fence and release/acquire flag crosses NVLink.
Skipped when fewer GPUs are visible than a test needs (the single-GPU
tests in test_rt.py / test_mpi.py run the same code paths with processes
sharing one device).

* halo DIRECT and FUSED_ASYNC at 2x1x1 and 2x2x2, every ghost cell verified
  (halo.hpp:237-254, 264-285);
* Send/Recv with every method and the model's choice, 1 KiB - 64 MiB,
  receiver bytes against the oracle;
* the NCCL baseline (batch pack, ncclSend/ncclRecv, batch unpack) verified
  like the engine's own exchange;
* neighbour alltoallw with layouts alternating across distinct devices.
"""
import os
import socket

import numpy as np
import pytest

from test_rt import _spawn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


def need_gpus(n):
    return pytest.mark.skipif(_ngpus() < n, reason=f"needs {n} visible GPUs (one process per device)")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _halo_distinct(rank, world, job, grid, method):
    import torch
    import paper_2012_14363_b200.halo as H
    import paper_2012_14363_b200.rt as rt
    torch.cuda.set_device(rank)
    rt.init(rank, world, job, device=rank, window_bytes=1 << 20, host_bytes=1 << 20)
    cfg = H.HaloConfig(grid, (24, 20, 16), 2, 32)
    alloc = torch.empty(28 * 24 * 20 * 32, dtype=torch.uint8, device="cuda")
    bad = 0
    for rnd in range(2):
        H.fill(cfg, rank, alloc)
        torch.cuda.synchronize()
        rt.barrier()
        plan = rt.HaloPlan(cfg, alloc, method)
        for _ in range(5):
            plan.exchange(timed=(rnd == 0))  # round 1: enqueue only (device-ordered iterations)
        torch.cuda.ExternalStream(rt.stream()).synchronize()
        bad += H.verify(cfg, rank, alloc)
        plan.free()
    rt.finalize()
    return bad


@pytest.mark.gpu
@pytest.mark.parametrize("method", [3, 2], ids=["direct", "fused_async"])
@pytest.mark.parametrize("grid", [(2, 1, 1), (2, 2, 2)])
def test_halo_on_distinct_devices(cuda, grid, method):
    world = grid[0] * grid[1] * grid[2]
    if _ngpus() < world:
        pytest.skip(f"needs {world} visible GPUs")
    assert set(_spawn(_halo_distinct, world, grid, method, timeout=300).values()) == {0}


def _cfg4_prog(e0, n):
    from tools.bench_parts import cfg4_prog
    return cfg4_prog(e0, n)


def _send_distinct(rank, world, job):
    import torch
    import paper_2012_14363_b200 as sp
    import paper_2012_14363_b200.model as M
    import paper_2012_14363_b200.rt as rt
    from oracle.pyoracle import oracle
    torch.cuda.set_device(rank)
    rt.init(rank, world, job, device=rank, window_bytes=80 << 20, host_bytes=80 << 20)
    rt.set_profile(M.load_profile_file(M.DEFAULT_B200_PROFILE))
    orc = oracle()
    methods = [rt.DEVICE, rt.ONESHOT, rt.STAGED, rt.DIRECT, rt.AUTO]
    used, bad, tag = [], 0, 0
    for e0 in (8, 64, 512):
        for n in (1 << 10, 1 << 14, 1 << 18, 1 << 22, 1 << 26):
            if n < 4 * e0:
                continue
            prog = _cfg4_prog(e0, n)
            ct = sp.commit_type(sp.from_program(prog))
            host = np.random.default_rng(e0 * 7 + n).integers(0, 256, ct.span, dtype=np.uint8)
            for m in methods:
                tag += 1
                if rank == 0:
                    used.append(rt.send(torch.from_numpy(host).cuda(), 1, ct, 1, tag=tag, method=m))
                else:
                    dst = torch.full((ct.span,), 0x3C, dtype=torch.uint8, device="cuda")
                    st = rt.recv(dst, 1, ct, source=0, tag=tag)
                    packed = np.zeros(ct.size, np.uint8)
                    orc.pack(prog, host, 1, packed, 0)
                    want = np.full(ct.span, 0x3C, np.uint8)
                    orc.unpack(prog, packed, 0, 1, want)
                    if not np.array_equal(dst.cpu().numpy(), want):
                        bad += 1
                    used.append(st["method"])
    rt.finalize()
    return bad, used


@pytest.mark.gpu
@need_gpus(2)
def test_send_every_method_on_distinct_devices(cuda):
    res = _spawn(_send_distinct, 2, timeout=600)
    assert res[1][0] == 0
    # the receiver saw the forced methods it was sent (DIRECT on device buffers)
    rx = res[1][1]
    assert rx[0::5] == [1] * len(rx[0::5]) and rx[3::5] == [3] * len(rx[3::5])


def _nccl_halo_distinct(rank, world, job, port):
    import torch
    import torch.distributed as dist
    import paper_2012_14363_b200.halo as H
    from tools.bench_parts import _nccl_halo, GRIDS
    torch.cuda.set_device(rank)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    cfg = H.HaloConfig(GRIDS[world], (24, 20, 16), 2, 32)
    regions = H.build_halo_types(cfg)
    seg = [0]
    for r in regions:
        seg.append(seg[-1] + r.send.size)
    alloc = torch.empty(28 * 24 * 20 * 32, dtype=torch.uint8, device="cuda")
    out = _nccl_halo(torch, cfg, regions, seg, alloc, rank, world, 3, 1, lambda i, s=None: None)
    dist.destroy_process_group()
    return out["verified"]


@pytest.mark.gpu
@need_gpus(2)
def test_nccl_halo_baseline_on_distinct_devices(cuda):
    assert all(_spawn(_nccl_halo_distinct, 2, _free_port(), timeout=300).values())


def _alternating_distinct(rank, world, job):
    """test_rt's alternating-layout regression, one device per rank"""
    import torch
    import test_rt
    real = torch.cuda.set_device
    torch.cuda.set_device = lambda d: real(rank)
    import paper_2012_14363_b200.rt as rt
    init = rt.init
    rt.init = lambda r, w, j, device=0, **kw: init(r, w, j, device=rank, **kw)
    return test_rt._nbr_alternating_layouts(rank, world, job, 200)


@pytest.mark.gpu
@need_gpus(3)
def test_neighbor_alltoallw_alternating_layouts_on_distinct_devices(cuda):
    res = _spawn(_alternating_distinct, 3, timeout=600)
    assert all(bad == 0 for bad, _ in res.values()), res
