"""The N>1 host path of bench.py on CPU: two ranks over torch.distributed
(gloo) agree on the max/sum reductions and on the runtime job name, then
bring up the engine's node-local runtime under that name (control plane
only, no GPU) and pass its barrier -- the same sequence the 2/4/8-GPU
scaling run executes with NCCL."""
import os
import socket
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    try:
        import torch
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import bench
        mx = bench.barrier_max(torch, world, float(rank + 1))
        sm = bench.barrier_sum(torch, world, float(rank + 1))
        job = bench.shared_job_name(world, rank)
        import paper_2012_14363_b200.rt as rt
        rt.init(rank, world, job, device=-1)
        for _ in range(50):
            rt.barrier()
        rt.finalize()
        dist.destroy_process_group()
        q.put((rank, mx, sm, job))
    except Exception as e:  # surfaced by the parent
        q.put((rank, "error", repr(e), None))


def test_bench_distributed_plumbing_gloo():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=180) for _ in range(2)]
    for p in ps:
        p.join(timeout=30)
    for r, mx, sm, job in out:
        assert mx != "error", sm
        assert mx == 2.0 and sm == 3.0
    assert out[0][3] == out[1][3]  # one job name for both ranks
