"""One pack and one unpack of cfg2 (K=64 objects) per E0 in {32, 64, 128,
512}, plus a dense 64 MiB copy as the streaming reference, each after an L2
flush -- the launches `scripts/gpu_r02_counters.sh` captures with ncu for the
DRAM counter table in profiles/r02_e0_counters.md."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2012_14363_b200 as sp  # noqa: E402

K = 64
torch.cuda.set_device(0)
src = torch.empty(K << 30, dtype=torch.uint8, device="cuda")
packed = torch.zeros(K << 20, dtype=torch.uint8, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
dense_a = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
dense_b = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")


def cold():
    flush.fill_(1)
    flush.view(torch.int64).sum()


def prog(e0):
    e2 = 2 ** math.ceil(math.log2((1 << 20) // e0) / 2)
    e1 = (1 << 20) // (e0 * e2)
    return [4, 3, 0, 1024, 1024, 1024, e0, e1, e2, 0, 0, 0, 0, 0]


for e0 in (32, 64, 128, 512):
    ct = sp.commit_type(sp.from_program(prog(e0)))
    cold()
    sp.pack(src, ct, K, packed, 0)
    cold()
    sp.unpack(packed, 0, ct, K, src)
cold()
dense_b.copy_(dense_a)
torch.cuda.synchronize()
print("done")
