"""One pack (or unpack) of an irregular hindexed byte type (mean block
--block bytes, ~64 MiB) for an ncu capture of the run-table kernel:
  ncu --set full -k regex:k_runs -c 1 python scripts/prof_runs.py --block 1024"""
import argparse
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2012_14363_b200 as sp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--block", type=int, default=1024)
ap.add_argument("--mode", choices=["pack", "unpack"], default="pack")
a = ap.parse_args()
rng = np.random.default_rng(1)
L, total = a.block, 64 << 20
n = total // L
lens = (rng.integers(L // 32, 3 * L // 32 + 1, n).clip(1) * 16).astype(np.int64)
gaps = (rng.integers(0, L // 16 + 1, n) * 16).astype(np.int64)
displs = np.cumsum(gaps + lens) - lens
perm = rng.permutation(n)
t = sp.commit_type(sp.make_hindexed(lens[perm].tolist(), displs[perm].tolist(), sp.make_named(sp.NamedKind.Byte)))
src = torch.randint(0, 256, (t.span,), dtype=torch.uint8, device="cuda")
dst = torch.empty(t.size, dtype=torch.uint8, device="cuda")
if a.mode == "pack":
    sp.pack(src, t, 1, dst, 0)
else:
    sp.unpack(dst, 0, t, 1, src)
torch.cuda.synchronize()
print(t.size, sp.last_launch())
