"""cfg1 = vector(131072,1,64,DOUBLE): one pack + one unpack of 1 object and
of 64 objects, each after an L2 flush -- the launches ncu captures for the
cfg1 sector-efficiency evidence (profiles/r02_cfg1_ncu.md)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2012_14363_b200 as sp  # noqa: E402

torch.cuda.set_device(0)
ct = sp.commit_type(sp.from_program([2, 131072, 1, 64, 0, 3]))
n = 64
src = torch.empty((n - 1) * ct.extent + ct.span, dtype=torch.uint8, device="cuda")
packed = torch.zeros(n * ct.size, dtype=torch.uint8, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for k in (1, n):
    for pack in (True, False):
        flush.fill_(1)
        flush.view(torch.int64).sum()
        if pack:
            sp.pack(src, ct, k, packed, 0)
        else:
            sp.unpack(packed, 0, ct, k, src)
torch.cuda.synchronize()
print("done")
