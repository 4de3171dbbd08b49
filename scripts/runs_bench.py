"""Run-table kernel (irregular indexed types) vs the strided kernels on the
same byte pattern: GB/s of pack and unpack, cold L2, CUDA events.

For each mean block length L, an irregular hindexed type of byte blocks
(lengths L/2..3L/2 rounded to 16, random gaps, scrambled definition order)
describing ~64 MiB, and the regular vector with the same L at the same
mean pitch (which the engine canonicalises to the strided kernels).

--misaligned: byte-granular lengths and gaps instead (word 1), the automatic
choice (k_runs_shift from 32-B mean runs) against the plain run kernel
forced with kernel=BlockList, at the same mean lengths."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2012_14363_b200 as sp  # noqa: E402


def timed(fn, flush, reps=5):
    ts = []
    for _ in range(reps):
        flush.fill_(1)  # 512 MiB written, then read back: a cold, clean L2
        flush.view(torch.int64).sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return sorted(ts)[len(ts) // 2]


def misaligned(flush):
    B = sp.make_named(sp.NamedKind.Byte)
    rng = np.random.default_rng(2)
    for L in (16, 32, 64, 256, 1024, 4096):
        n = (64 << 20) // L
        lens = rng.integers(max(1, L // 2), 3 * L // 2 + 1, n).astype(np.int64)
        gaps = rng.integers(0, L + 1, n).astype(np.int64)
        displs = np.cumsum(gaps + lens) - lens + 3
        perm = rng.permutation(n)
        t = sp.commit_type(sp.make_hindexed(lens[perm].tolist(), displs[perm].tolist(), B))
        src = torch.randint(0, 256, (t.span,), dtype=torch.uint8, device="cuda")
        dst = torch.empty(t.size, dtype=torch.uint8, device="cuda")
        row = {"mean_block": L, "runs": int(n), "bytes": int(t.size), "misaligned": True}
        row["auto_pack_us"] = timed(lambda: sp.pack(src, t, 1, dst, 0), flush)
        row["auto_word"] = sp.last_launch().word
        row["auto_unpack_us"] = timed(lambda: sp.unpack(dst, 0, t, 1, src), flush)
        row["plain_pack_us"] = timed(lambda: sp.pack(src, t, 1, dst, 0, kernel=sp.Kernel.BlockList), flush)
        row["plain_word"] = sp.last_launch().word
        row["plain_unpack_us"] = timed(lambda: sp.unpack(dst, 0, t, 1, src, kernel=sp.Kernel.BlockList), flush)
        for k in ("auto_pack", "auto_unpack", "plain_pack", "plain_unpack"):
            row[k + "_GBps"] = round(2 * t.size / row[k + "_us"] / 1e3, 1)
        print(json.dumps(row), flush=True)
        del src, dst


def main():
    torch.cuda.set_device(0)
    if "--misaligned" in sys.argv:
        misaligned(torch.empty(512 << 20, dtype=torch.uint8, device="cuda"))
        return
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    B = sp.make_named(sp.NamedKind.Byte)
    rng = np.random.default_rng(1)
    out = []
    for L in (16, 64, 256, 1024, 4096):
        total = 64 << 20
        n = total // L
        lens = (rng.integers(L // 32, 3 * L // 32 + 1, n).clip(1) * 16).astype(np.int64)
        gaps = (rng.integers(0, L // 16 + 1, n) * 16).astype(np.int64)
        displs = np.cumsum(gaps + lens) - lens
        perm = rng.permutation(n)
        t = sp.commit_type(sp.make_hindexed(lens[perm].tolist(), displs[perm].tolist(), B))
        assert t.form == sp.CanonForm.Unsupported
        src = torch.randint(0, 256, (t.span,), dtype=torch.uint8, device="cuda")
        dst = torch.empty(t.size, dtype=torch.uint8, device="cuda")
        pitch = int(np.mean(gaps + lens)) // 16 * 16
        v = sp.commit_type(sp.make_hvector(total // L, L, pitch, B))
        vsrc = torch.randint(0, 256, (v.span,), dtype=torch.uint8, device="cuda")
        vdst = torch.empty(v.size, dtype=torch.uint8, device="cuda")
        row = {"mean_block": L, "runs": int(n), "bytes": int(t.size)}
        row["runs_pack_us"] = timed(lambda: sp.pack(src, t, 1, dst, 0), flush)
        row["runs_word"] = sp.last_launch().word
        row["runs_unpack_us"] = timed(lambda: sp.unpack(dst, 0, t, 1, src), flush)
        row["strided_pack_us"] = timed(lambda: sp.pack(vsrc, v, 1, vdst, 0), flush)
        row["strided_unpack_us"] = timed(lambda: sp.unpack(vdst, 0, v, 1, vsrc), flush)
        for k in ("runs_pack", "runs_unpack", "strided_pack", "strided_unpack"):
            nbytes = t.size if k.startswith("runs") else v.size
            row[k + "_GBps"] = round(2 * nbytes / row[k + "_us"] / 1e3, 1)
        out.append(row)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
