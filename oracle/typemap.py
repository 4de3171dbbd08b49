"""MPI-3.1 typemap restatement -- TEST INFRASTRUCTURE ONLY (imported by tests/,
never by the product path).

No reference vectors: the reference has no indexed, struct or resized
datatypes (PAPER.md:1164 lists them as future
work). Pinned instead to an external source: the worked typemap examples of
the MPI-3.1 standard (section 4.1.2: contiguous, vector, indexed, struct),
transcribed in tests/golden/mpi31_typemap_examples.json and checked by
tests/test_mpi31_examples.py against this module AND the engine. This module restates the
MPI-3.1 definitions directly (sections 4.1.2 contiguous, 4.1.3 vector and
hvector, 4.1.4 indexed/hindexed, 4.1.5 indexed_block/hindexed_block, 4.1.6
struct, 4.1.7 resized, 4.1.3 subarray) in pure Python, small sizes only:

* the typemap in definition order as byte runs (offset, length), adjacent
  runs coalesced -- the order the engine packs block-list forms in;
* size, lb and extent (no alignment padding for struct, as documented for
  the engine; negative displacements are outside the engine's domain).

A type description is a nested tuple:
  ("named", nbytes)
  ("contiguous", n, inner)
  ("vector", count, blocklength, stride_in_inner_extents, inner)
  ("hvector", count, blocklength, stride_bytes, inner)
  ("subarray", sizes, subsizes, offsets, inner)        dim 0 innermost
  ("indexed", blocklengths, displs_in_inner_extents, inner)
  ("hindexed", blocklengths, displs_bytes, inner)
  ("struct", blocklengths, displs_bytes, [members])
  ("resized", lb, extent, inner)
"""


def _push(out, off, n):
    if n == 0:
        return
    if out and out[-1][0] + out[-1][1] == off:
        out[-1] = (out[-1][0], out[-1][1] + n)
    else:
        out.append((off, n))


def _place(out, runs, base):
    for off, n in runs:
        _push(out, base + off, n)


def typemap(d):
    """(size, lb, extent, runs in definition order) of description d"""
    k = d[0]
    if k == "named":
        n = d[1]
        return n, 0, n, [(0, n)]
    if k == "contiguous":
        n, inner = d[1], d[2]
        s, lb, ext, r = typemap(inner)
        out = []
        for i in range(n):
            _place(out, r, i * ext)
        return n * s, (lb if n else 0), n * ext, out
    if k in ("vector", "hvector"):
        c, bl, st, inner = d[1:]
        s, lb, ext, r = typemap(inner)
        step = st * ext if k == "vector" else st
        out = []
        for i in range(c):
            for j in range(bl):
                _place(out, r, i * step + j * ext)
        if c == 0 or bl == 0:
            return 0, 0, 0, out
        # MPI: the blocks' lower/upper bounds; strides are nonnegative here
        return c * bl * s, lb, (c - 1) * step + bl * ext, out
    if k == "subarray":
        sizes, subsizes, offsets, inner = d[1:]
        s, lb, ext, r = typemap(inner)
        nd = len(sizes)
        dstride, acc = [], ext
        for i in range(nd):
            dstride.append(acc)
            acc *= sizes[i]
        out = []
        idx = [0] * nd
        while True:
            _place(out, r, sum((offsets[i] + idx[i]) * dstride[i] for i in range(nd)))
            i = 0
            while i < nd:
                idx[i] += 1
                if idx[i] < subsizes[i]:
                    break
                idx[i] = 0
                i += 1
            if i == nd:
                break
        n = 1
        for x in subsizes:
            n *= x
        return n * s, 0, acc, out
    if k in ("indexed", "hindexed", "struct"):
        bls, displs = d[1], d[2]
        members = d[3] if k == "struct" else [d[3]] * len(bls)
        out, size, lo, hi = [], 0, None, None
        for bl, disp, m in zip(bls, displs, members):
            s, lb, ext, r = typemap(m)
            byte_disp = disp * ext if k == "indexed" else disp
            for j in range(bl):
                _place(out, r, byte_disp + j * ext)
            size += bl * s
            if bl:
                a, b = byte_disp + lb, byte_disp + lb + bl * ext
                lo = a if lo is None else min(lo, a)
                hi = b if hi is None else max(hi, b)
        if lo is None:
            return size, 0, 0, out
        return size, lo, hi - lo, out
    if k == "resized":
        lb, ext, inner = d[1:]
        s, _, _, r = typemap(inner)
        return s, lb, ext, list(r)
    raise ValueError(f"unknown constructor {k}")


def normalized(runs):
    """sorted, abutting/overlapping runs merged; (runs, overlap)"""
    out, overlap = [], False
    for off, n in sorted(runs):
        if out and off <= out[-1][0] + out[-1][1]:
            if off < out[-1][0] + out[-1][1]:
                overlap = True
            end = max(out[-1][0] + out[-1][1], off + n)
            out[-1] = (out[-1][0], end - out[-1][0])
        else:
            out.append((off, n))
    return out, overlap


def span(runs):
    return max((o + n for o, n in runs), default=0)


def gather(src, runs, count, extent, size):
    """packed bytes of `count` objects, runs in the given order"""
    import numpy as np
    out = np.empty(count * size, np.uint8)
    p = 0
    for j in range(count):
        for off, n in runs:
            out[p:p + n] = src[j * extent + off:j * extent + off + n]
            p += n
    assert p == count * size
    return out


def scatter(packed, dst, runs, count, extent):
    p = 0
    for j in range(count):
        for off, n in runs:
            dst[j * extent + off:j * extent + off + n] = packed[p:p + n]
            p += n
    return dst


def build(sp, d):
    """the engine's definition of description d (through the public API)"""
    k = d[0]
    named = {1: sp.NamedKind.Byte, 4: sp.NamedKind.Int, 8: sp.NamedKind.Double}
    if k == "named":
        return sp.make_named(named[d[1]])
    if k == "contiguous":
        return sp.make_contiguous(d[1], build(sp, d[2]))
    if k == "vector":
        return sp.make_vector(d[1], d[2], d[3], build(sp, d[4]))
    if k == "hvector":
        return sp.make_hvector(d[1], d[2], d[3], build(sp, d[4]))
    if k == "subarray":
        return sp.make_subarray(len(d[1]), d[1], d[2], d[3], build(sp, d[4]))
    if k == "indexed":
        return sp.make_indexed(d[1], d[2], build(sp, d[3]))
    if k == "hindexed":
        return sp.make_hindexed(d[1], d[2], build(sp, d[3]))
    if k == "struct":
        return sp.make_struct(d[1], d[2], [build(sp, m) for m in d[3]])
    if k == "resized":
        return sp.make_resized(build(sp, d[3]), d[1], d[2])
    raise ValueError(k)


def random_desc(rng, depth=0):
    """a random description with a small span (a few KiB at most)"""
    leaves = [("named", 1), ("named", 4), ("named", 8)]
    if depth >= 3 or rng.random() < 0.25:
        return leaves[int(rng.integers(0, 3))]
    inner = random_desc(rng, depth + 1)
    _, _, ext, _ = typemap(inner)
    ext = max(ext, 1)
    k = int(rng.integers(0, 8))
    if k == 0:
        return ("contiguous", int(rng.integers(1, 4)), inner)
    if k == 1:
        bl = int(rng.integers(1, 3))
        return ("vector", int(rng.integers(1, 4)), bl, bl + int(rng.integers(0, 3)), inner)
    if k == 2:
        n = int(rng.integers(1, 6))
        bls = [int(rng.integers(0, 3)) for _ in range(n)]
        ds = sorted(int(x) for x in rng.choice(4 * n + 4, n, replace=False))
        if rng.random() < 0.3:
            ds = ds[::-1]  # decreasing displacements: typemap order != address order
        return ("indexed", bls, ds, inner)
    if k == 3:
        n = int(rng.integers(1, 6))
        bls = [int(rng.integers(1, 3))] * n if rng.random() < 0.5 else [int(rng.integers(0, 4)) for _ in range(n)]
        step = int(rng.integers(0, 3)) * ext + int(rng.integers(0, 9)) * (ext if rng.random() < 0.5 else 1)
        ds = [i * max(step, 1) + (int(rng.integers(0, 5)) if rng.random() < 0.3 else 0) for i in range(n)]
        return ("hindexed", bls, ds, inner)
    if k == 4:
        n = int(rng.integers(1, 4))
        members = [inner] + [random_desc(rng, depth + 2) for _ in range(n - 1)]
        ds, at = [], 0
        bls = []
        for m in members:
            _, _, e, _ = typemap(m)
            bl = int(rng.integers(1, 3))
            at += int(rng.integers(0, 9))
            ds.append(at)
            bls.append(bl)
            at += bl * max(e, 1)
        return ("struct", bls, ds, members)
    if k == 5:
        return ("resized", 0, ext + int(rng.integers(0, 2 * ext + 1)), inner)
    if k == 6:
        return ("hvector", int(rng.integers(1, 4)), int(rng.integers(1, 3)),
                int(rng.integers(0, 3)) * ext + int(rng.integers(1, 3 * ext + 2)), inner)
    nd = int(rng.integers(1, 3))
    sizes = [int(rng.integers(1, 5)) for _ in range(nd)]
    sub = [int(rng.integers(1, s + 1)) for s in sizes]
    offs = [int(rng.integers(0, s - b + 1)) for s, b in zip(sizes, sub)]
    return ("subarray", sizes, sub, offs, inner)
