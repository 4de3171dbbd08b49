"""e2e variants (bench.py's e2e leg): device time per step for messages of
Ke/split objects per E0 in three issue orders over NS streams, and the PCIe
bound (the same bytes as plain copies in both directions at once). Measured
on B200 (round 1): every variant 2.30-2.71 ms against a 1.71 ms bound; the
same loop driven from C++ instead of Python was within noise (2.26-2.43)."""
import ctypes as C, math, os, sys, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2012_14363_b200 as sp
from paper_2012_14363_b200 import _capi
lib = _capi.lib
E0S = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512]
def prog(e0):
    e2 = 2 ** math.ceil(math.log2((1 << 20) // e0) / 2)
    e1 = (1 << 20) // (e0 * e2)
    return [4, 3, 0, 1024, 1024, 1024, e0, e1, e2, 0, 0, 0, 0, 0]
types = [(e0, sp.commit_type(sp.from_program(prog(e0)))) for e0 in E0S]
Ke = 8
xoff, at = {}, 0
for e0 in sorted(E0S, reverse=True):
    xoff[e0] = at; at += e0
esrc = torch.empty((Ke << 30) + 4096, dtype=torch.uint8, device="cuda")
msg_in = [torch.full((Ke << 20,), 5, dtype=torch.uint8).pin_memory() for _ in E0S]
msg_out = [torch.empty(Ke << 20, dtype=torch.uint8).pin_memory() for _ in E0S]
pos = C.c_int64(0)
res = {}
ORDERS = {"desc": sorted(E0S, reverse=True), "asc": sorted(E0S), "mix": [1, 4, 8, 16, 2, 32, 64, 128, 256, 512]}
idx = {e0: i for i, (e0, _) in enumerate(types)}


def pieces(splits):
    """messages as (e0, first object, objects), the slow small-E0 objects
    split finer and dealt between the fast ones"""
    fast = [(e0, j, Ke // splits.get(e0, 1)) for e0 in sorted(E0S, reverse=True)
            for j in range(0, Ke, Ke // splits.get(e0, 1)) if splits.get(e0, 1) == 1]
    slow = [(e0, j, Ke // splits[e0]) for e0 in sorted(E0S) if splits.get(e0, 1) > 1
            for j in range(0, Ke, Ke // splits[e0])]
    out = []
    while fast or slow:
        if fast:
            out.append(fast.pop(0))
        for _ in range(max(1, len(slow) // max(1, len(fast) + 1))):
            if slow:
                out.append(slow.pop(0))
    return out


VARIANTS = [(10, "per-E0 desc", [(e0, 0, Ke) for e0 in ORDERS["desc"]]),
            (16, "split E0<=4 x8", pieces({1: 8, 2: 8, 4: 8})),
            (16, "split E0<=8 x4", pieces({1: 4, 2: 4, 4: 4, 8: 4})),
            (24, "split E0<=16 x8", pieces({1: 8, 2: 8, 4: 8, 8: 8, 16: 8})),
            (8, "split E0<=4 x8 NS8", pieces({1: 8, 2: 8, 4: 8}))]
for NS, label, msgs in VARIANTS:
    streams = [torch.cuda.Stream() for _ in range(NS)]
    handles = (C.c_void_p * NS)(*[s.cuda_stream for s in streams])
    items = []
    for e0, j0, per in msgs:
        i = idx[e0]
        ct = types[i][1]
        items.append((ct, esrc.data_ptr() + (j0 << 30) + xoff[e0], msg_in[i].data_ptr() + (j0 << 20),
                      msg_out[i].data_ptr() + (j0 << 20), per << 20, per))
    per_obj = label
    n = len(items)
    arr_t = (_capi.sp_type * n)(*[it[0].handle for it in items])
    arr_c = (C.c_int64 * n)(*[it[5] for it in items])
    arr_o = (C.c_void_p * n)(*[it[1] for it in items])
    arr_ob = (C.c_uint64 * n)(*[esrc.numel() - (it[1] - esrc.data_ptr()) for it in items])
    arr_i = (C.c_void_p * n)(*[it[2] for it in items])
    arr_out = (C.c_void_p * n)(*[it[3] for it in items])
    arr_mb = (C.c_uint64 * n)(*[it[4] for it in items])
    dev, host = [], []
    for it in range(8):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(streams[0])
        for s in streams[1:]: s.wait_event(a)
        t0 = time.perf_counter()
        for k, (ct, obj, mi, mo, mb, cnt) in enumerate(items):
            h = C.c_void_p(handles[k % NS])
            pos.value = 0
            assert lib.sp_unpack(mi, mb, C.byref(pos), ct.handle, cnt, obj, esrc.numel(), h) == 0
            pos.value = 0
            assert lib.sp_pack(obj, esrc.numel(), ct.handle, cnt, mo, mb, C.byref(pos), h) == 0
        t1 = time.perf_counter()
        for s in streams[1:]:
            ev = torch.cuda.Event(); ev.record(s); streams[0].wait_event(ev)
        b.record(streams[0])
        torch.cuda.synchronize()
        if it >= 3:
            dev.append(a.elapsed_time(b)); host.append((t1 - t0) * 1e3)
    bytes_ = 2 * Ke * (1 << 20) * 2 * len(E0S)
    res[f"NS={NS} {per_obj}"] = {"dev_ms": round(min(dev), 3), "host_ms": round(min(host), 3),
                                                         "GBps": round(bytes_ / (min(dev) * 1e-3) / 1e9, 1)}
# PCIe bound
dev_buf = torch.empty(2 * (Ke << 20) * len(E0S), dtype=torch.uint8, device="cuda")
hin = torch.cat(msg_in).pin_memory()
hout = torch.empty_like(hin).pin_memory()
half = hin.numel()
s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
pc = []
for it in range(5):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s0); s1.wait_event(a)
    with torch.cuda.stream(s0): dev_buf[:half].copy_(hin, non_blocking=True)
    with torch.cuda.stream(s1): hout.copy_(dev_buf[half:], non_blocking=True)
    ev = torch.cuda.Event(); ev.record(s1); s0.wait_event(ev); b.record(s0)
    torch.cuda.synchronize()
    if it: pc.append(a.elapsed_time(b))
res["pcie_bound_ms"] = round(min(pc), 3)
print(json.dumps(res, indent=1))
