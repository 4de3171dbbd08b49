"""One launch of every kernel the automatic choice uses, each after an L2
flush, for an ncu counter pass (scripts/gpu_kernel_choices.sh): the
north star asks for every kernel choice to be backed by counters (achieved
HBM GB/s and sector efficiency).

Launch order (the table script relies on it):
  cfg2 E0 = 1..512, K = 64: pack, unpack           (20 launches)
  cfg1 vector(131072,1,64,DOUBLE), K = 64: pack, unpack  (2)
  misaligned subarray (rows of 256 B, start at byte 3), K = 16: pack, unpack (2)
  irregular hindexed, ~64 MiB, mean block 1 KiB, byte-aligned: pack, unpack  (2)
  the same rounded to 16 B: pack, unpack  (2)
  halo 256^3 r=2 32 B, one rank: the DIRECT typed-copy batch  (1)
Each line printed: index, label, algorithmic bytes, kernel/word chosen.
"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_14363_b200 as sp  # noqa: E402
import paper_2012_14363_b200.halo as H  # noqa: E402


def cfg2(e0):
    e2 = 2 ** math.ceil(math.log2((1 << 20) // e0) / 2)
    e1 = (1 << 20) // (e0 * e2)
    return [4, 3, 0, 1024, 1024, 1024, e0, e1, e2, 0, 0, 0, 0, 0]


def main():
    torch.cuda.set_device(0)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    idx = [0]

    def run(label, nbytes, fn):
        flush.fill_(1)
        torch.sum(flush.view(torch.int64))
        torch.cuda.synchronize()
        fn()
        torch.cuda.synchronize()
        li = sp.last_launch()
        print(f"{idx[0]}\t{label}\t{nbytes}\t{li.kernel.name}/w{li.word}", flush=True)
        idx[0] += 1

    K = 64
    big = torch.empty(K << 30, dtype=torch.uint8, device="cuda")
    big[::4099] = 3
    packed = torch.zeros(K << 20, dtype=torch.uint8, device="cuda")
    for e0 in (1, 2, 4, 8, 16, 32, 64, 128, 256, 512):
        ct = sp.commit_type(sp.from_program(cfg2(e0)))
        run(f"cfg2 E0={e0} pack", 2 * K * ct.size, lambda: sp.pack(big, ct, K, packed, 0))
        run(f"cfg2 E0={e0} unpack", 2 * K * ct.size, lambda: sp.unpack(packed, 0, ct, K, big))
    ct = sp.commit_type(sp.from_program([2, 131072, 1, 64, 0, 3]))
    run("cfg1 pack", 2 * K * ct.size, lambda: sp.pack(big, ct, K, packed, 0))
    run("cfg1 unpack", 2 * K * ct.size, lambda: sp.unpack(packed, 0, ct, K, big))
    del big
    # rows of 256 B starting at byte 3: addresses force W = 1, the shift kernels
    sub = sp.commit_type(sp.make_subarray(3, [1024, 1024, 1024], [256, 64, 256], [3, 0, 0],
                                          sp.make_named(sp.NamedKind.Byte)))
    src = torch.empty(16 * sub.extent, dtype=torch.uint8, device="cuda")
    dst = torch.zeros(16 * sub.size, dtype=torch.uint8, device="cuda")
    run("misaligned 256-B rows pack", 2 * 16 * sub.size, lambda: sp.pack(src, sub, 16, dst, 0))
    run("misaligned 256-B rows unpack", 2 * 16 * sub.size, lambda: sp.unpack(dst, 0, sub, 16, src))
    del src, dst
    # irregular hindexed: 65536 blocks of 512-1536 B at random gaps
    rng = np.random.default_rng(5)
    bl = rng.integers(512, 1537, 65536)
    disp = np.concatenate([[0], np.cumsum(bl + rng.integers(16, 2048, 65536))[:-1]])
    it = sp.commit_type(sp.make_hindexed([int(x) for x in bl], [int(x) for x in disp],
                                         sp.make_named(sp.NamedKind.Byte)))
    src = torch.empty(it.span, dtype=torch.uint8, device="cuda")
    dst = torch.zeros(it.size, dtype=torch.uint8, device="cuda")
    run("irregular hindexed 1 KiB, byte-aligned pack", 2 * it.size, lambda: sp.pack(src, it, 1, dst, 0))
    run("irregular hindexed 1 KiB, byte-aligned unpack", 2 * it.size, lambda: sp.unpack(dst, 0, it, 1, src))
    del src, dst
    # the same sizes rounded to 16 B: the plain run kernel at word 16
    bl16 = (bl + 15) // 16 * 16
    d16 = np.concatenate([[0], np.cumsum(bl16 + rng.integers(1, 128, 65536) * 16)[:-1]])
    it = sp.commit_type(sp.make_hindexed([int(x) for x in bl16], [int(x) for x in d16],
                                         sp.make_named(sp.NamedKind.Byte)))
    src = torch.empty(it.span, dtype=torch.uint8, device="cuda")
    dst = torch.zeros(it.size, dtype=torch.uint8, device="cuda")
    run("irregular hindexed 1 KiB, 16-B aligned pack", 2 * it.size, lambda: sp.pack(src, it, 1, dst, 0))
    run("irregular hindexed 1 KiB, 16-B aligned unpack", 2 * it.size, lambda: sp.unpack(dst, 0, it, 1, src))
    del src, dst
    # halo DIRECT at one rank: the 26 region types as one typed-copy batch
    cfg = H.HaloConfig((1, 1, 1), (256, 256, 256), 2, 32)
    regions = H.build_halo_types(cfg)
    pad = 260 ** 3 * 32
    alloc = torch.empty(pad, dtype=torch.uint8, device="cuda")
    b = H.Batch.copies([(alloc, regions[j].send, 1, alloc, regions[25 - j].recv, 1) for j in range(26)])
    run("halo DIRECT copy batch", 2 * b.bytes, lambda: b.execute())


if __name__ == "__main__":
    main()
