"""e2e variants (bench.py's e2e leg): host time per step vs device time,
for NS streams and per-object vs per-E0 messages through the C-ABI."""
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
for NS, per_obj in [(4, True), (2, True), (8, True), (4, False), (10, False)]:
    streams = [torch.cuda.Stream() for _ in range(NS)]
    handles = [C.c_void_p(s.cuda_stream) for s in streams]
    items = []
    order = sorted(range(len(types)), key=lambda i: -types[i][0])
    if per_obj:
        for j in range(Ke):
            for i in order:
                items.append((types[i][1], esrc.data_ptr() + (j << 30) + xoff[types[i][0]], j << 20, i, 1))
    else:
        for i in order:
            items.append((types[i][1], esrc.data_ptr() + xoff[types[i][0]], 0, i, Ke))
    dev, host = [], []
    for it in range(8):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(streams[0])
        for s in streams[1:]: s.wait_event(a)
        t0 = time.perf_counter()
        for n, (ct, obj, off, i, cnt) in enumerate(items):
            h = handles[n % NS]
            pos.value = off
            assert lib.sp_unpack(msg_in[i].data_ptr(), msg_in[i].numel(), C.byref(pos), ct.handle, cnt, obj, esrc.numel(), h) == 0
            pos.value = off
            assert lib.sp_pack(obj, esrc.numel(), ct.handle, cnt, msg_out[i].data_ptr(), msg_out[i].numel(), C.byref(pos), h) == 0
        t1 = time.perf_counter()
        for s in streams[1:]:
            ev = torch.cuda.Event(); ev.record(s); streams[0].wait_event(ev)
        b.record(streams[0])
        torch.cuda.synchronize()
        if it >= 3:
            dev.append(a.elapsed_time(b)); host.append((t1 - t0) * 1e3)
    bytes_ = 2 * Ke * (1 << 20) * 2 * len(E0S)
    res[f"NS={NS} per_obj={per_obj}"] = {"dev_ms": round(min(dev), 3), "host_ms": round(min(host), 3),
                                         "GBps": round(bytes_ / (min(dev) * 1e-3) / 1e9, 1)}
print(json.dumps(res, indent=1))
