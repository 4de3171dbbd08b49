"""Datatypes beyond the reference: MPI indexed / hindexed / indexed_block /
struct / resized (MPI-3.1 4.1.2-4.1.7; PAPER.md:1164 lists them as TEMPI's
future work). The reference has none of them, so
parity rests on the MPI typemap restatement in oracle/typemap.py, which is
itself pinned to the MPI-3.1 standard's worked examples
(tests/test_mpi31_examples.py), not to reference vectors.

CPU: size / lb / extent / span / flattened runs / overlap against the
restatement over thousands of random nested descriptions, canonicalisation
of regular index patterns to StridedBlocks, and the sixth config-3
construction (vector of a resized hvector) that needed MPI_Type_create_resized.
GPU: pack and unpack parity of random descriptions (block-list forms in
typemap order, strided forms in the canonical order), and a large irregular
indexed type through the run-table kernel at every legal word size.
"""
import numpy as np
import pytest

from oracle import typemap as tm


def _runs(bl):
    return [(b.offset, b.length) for b in bl.blocks]


def test_random_descriptions_match_typemap(sp):
    rng = np.random.default_rng(5)
    forms = {0: 0, 2: 0}
    for _ in range(2000):
        d = tm.random_desc(rng)
        size, lb, ext, runs = tm.typemap(d)
        t = tm.build(sp, d)
        assert (t.size(), t.lb(), t.extent()) == (size, lb, ext), d
        norm, ov = tm.normalized(runs)
        fl = sp.flatten(t)
        assert _runs(fl) == norm and fl.overlap == ov, d
        if size == 0:
            continue
        c = sp.commit_type(t)
        forms[int(c.form)] += 1
        assert c.span == tm.span(runs), d
        if c.form == sp.CanonForm.Strided and not c.overlapping:
            assert _runs(sp.enumerate_blocks(c.canon)) == norm, d
        if c.form == sp.CanonForm.Unsupported:
            assert c.overlapping == ov, d
    assert forms[0] > 500 and forms[2] > 200


def test_regular_index_patterns_canonicalise(sp):
    D = sp.make_named(sp.NamedKind.Double)
    B = sp.make_named(sp.NamedKind.Byte)
    # equal blocks at an arithmetic progression == hvector
    c = sp.commit_type(sp.make_indexed([2, 2, 2], [0, 5, 10], D))
    assert c.form == sp.CanonForm.Strided
    assert c.canon == sp.StridedBlock(0, (16, 3), (1, 40))
    assert c.extent == 96
    # abutting blocks merge; an offset first block moves the start and lb
    t = sp.make_hindexed([3, 5], [64, 67], B)
    c = sp.commit_type(t)
    assert c.canon == sp.StridedBlock(64, (8,), (1,)) and t.lb() == 64 and c.extent == 8
    # indexed_block with a stride pattern == vector
    c = sp.commit_type(sp.make_indexed_block(4, [0, 16, 32, 48], sp.make_named(sp.NamedKind.Float)))
    assert c.canon == sp.StridedBlock(0, (16, 4), (1, 64))
    # a struct of one member type at a progression is strided too
    c = sp.commit_type(sp.make_struct([1, 1, 1], [0, 24, 48], [D, D, D]))
    assert c.canon == sp.StridedBlock(0, (8, 3), (1, 24))
    # irregular: block-list form, unpackable because nothing repeats
    c = sp.commit_type(sp.make_indexed([2, 3, 1], [1, 5, 10], D))
    assert c.form == sp.CanonForm.Unsupported and not c.overlapping
    # repeated bytes: block-list form that refuses unpack
    c = sp.commit_type(sp.make_hindexed([1, 1], [0, 0], D))
    assert c.overlapping


def test_struct_and_resized_bounds(sp):
    I = sp.make_named(sp.NamedKind.Int)
    D = sp.make_named(sp.NamedKind.Double)
    s = sp.make_struct([1, 2], [0, 8], [I, D])
    assert (s.size(), s.lb(), s.extent()) == (20, 0, 24)  # no alignment padding
    r = sp.make_resized(s, 0, 32)
    assert (r.size(), r.lb(), r.extent()) == (20, 0, 32)
    c = sp.commit_type(sp.make_contiguous(4, r))
    assert c.extent == 128 and c.span == 3 * 32 + 24
    r2 = sp.make_resized(D, -8, 16)
    assert r2.lb() == -8 and r2.extent() == 16
    c = sp.commit_type(sp.make_contiguous(3, sp.make_resized(D, 0, 16)))
    assert c.canon == sp.StridedBlock(0, (8, 3), (1, 16))


def test_config3_vector_of_resized_hvector(sp):
    """BASELINE config 3 notes that a true vector-of-hvector cuboid needs
    MPI_Type_create_resized: with it, the sixth construction reaches the same
    StridedBlock and plan as the subarray"""
    B = sp.make_named(sp.NamedKind.Byte)
    for e0, e1, e2 in [(32, 128, 256), (1, 1024, 1024), (512, 32, 64)]:
        col = sp.make_hvector(e1, 1, 1024, sp.make_contiguous(e0, B))
        six = sp.commit_type(sp.make_vector(e2, 1, 1, sp.make_resized(col, 0, 1 << 20)))
        sub = sp.commit_type(sp.make_subarray(3, [1024] * 3, [e0, e1, e2], [0, 0, 0], B))
        assert six.canon == sub.canon and six.plan == sub.plan


def test_constructor_errors(sp):
    D = sp.make_named(sp.NamedKind.Double)
    with pytest.raises(sp.InvalidArgument):
        sp.make_hindexed([1], [-8], D)
    with pytest.raises(sp.InvalidArgument):
        sp.make_indexed([-1], [0], D)
    with pytest.raises(sp.InvalidArgument):
        sp.make_resized(D, 0, -1)
    with pytest.raises(sp.InvalidArgument):
        sp.make_struct([1, 1], [0], [D, D])


# ------------------------------------------------------------ GPU parity
def _canonical_runs(sb):
    """the strided form's pack order: counts[0]-byte runs, dim 1 fastest"""
    import itertools
    dims = [range(c) for c in sb.counts[1:]]
    out = []
    for idx in itertools.product(*reversed(dims)):
        out.append((sb.start + sum(i * s for i, s in zip(reversed(idx), sb.strides[1:])), sb.counts[0]))
    return out


@pytest.mark.gpu
def test_random_descriptions_pack_unpack_gpu(sp, cuda):
    torch = cuda
    rng = np.random.default_rng(17)
    checked = {0: 0, 2: 0}
    for _ in range(600):
        d = tm.random_desc(rng)
        size, lb, ext, runs = tm.typemap(d)
        if size == 0:
            continue
        c = sp.commit_type(tm.build(sp, d))
        order = _canonical_runs(c.canon) if c.form == sp.CanonForm.Strided else runs
        inc = 1 + int(rng.integers(0, 3))
        pos = int(rng.integers(0, 9))
        span = (inc - 1) * c.extent + c.span
        host = rng.integers(0, 256, span, dtype=np.uint8)
        want = tm.gather(host, order, inc, c.extent, size)
        src = torch.from_numpy(host).cuda()
        dst = torch.full((pos + inc * size + 8,), 0xEE, dtype=torch.uint8, device="cuda")
        assert sp.pack(src, c, inc, dst, pos) == pos + inc * size
        got = dst.cpu().numpy()
        assert np.array_equal(got[pos:pos + inc * size], want), d
        assert (got[:pos] == 0xEE).all() and (got[pos + inc * size:] == 0xEE).all()
        if not c.overlapping:
            exp = tm.scatter(want, np.full(span, 0x5A, np.uint8), order, inc, c.extent)
            out = torch.full((span,), 0x5A, dtype=torch.uint8, device="cuda")
            sp.unpack(dst, pos, c, inc, out)
            assert np.array_equal(out.cpu().numpy(), exp), d
        checked[int(c.form)] += 1
    assert checked[0] > 150 and checked[2] > 50


@pytest.mark.gpu
@pytest.mark.parametrize("word", [0, 1, 2, 4, 8, 16])
def test_large_irregular_indexed_gpu(sp, cuda, word):
    """20,000 blocks of 16..4096 B (multiples of 16) at irregular
    displacements: the run-table kernel at its natural word (0 = auto, 16
    here) and every forced smaller word"""
    torch = cuda
    rng = np.random.default_rng(99)
    n = 20000
    bls = (rng.integers(1, 257, n) * 16).tolist()
    gaps = (rng.integers(0, 64, n) * 16).tolist()
    displs, at = [], 0
    for b, g in zip(bls, gaps):
        at += g
        displs.append(at)
        at += b
    perm = rng.permutation(n)  # typemap order differs from address order
    bls = [bls[i] for i in perm]
    displs = [displs[i] for i in perm]
    B = sp.make_named(sp.NamedKind.Byte)
    c = sp.commit_type(sp.make_hindexed(bls, displs, B))
    assert c.form == sp.CanonForm.Unsupported and not c.overlapping
    runs = list(zip(displs, bls))
    span = c.span
    host = rng.integers(0, 256, c.extent + span, dtype=np.uint8)
    want = tm.gather(host, runs, 2, c.extent, c.size)
    src = torch.from_numpy(host).cuda()
    dst = torch.empty(2 * c.size, dtype=torch.uint8, device="cuda")
    kw = dict(force_word=word) if word else {}
    sp.pack(src, c, 2, dst, 0, **kw)
    assert sp.last_launch().word == (word or 16)
    assert np.array_equal(dst.cpu().numpy(), want)
    out = torch.zeros(c.extent + span, dtype=torch.uint8, device="cuda")
    sp.unpack(dst, 0, c, 2, out, **kw)
    exp = tm.scatter(want, np.zeros(c.extent + span, np.uint8), runs, 2, c.extent)
    assert np.array_equal(out.cpu().numpy(), exp)


@pytest.mark.gpu
@pytest.mark.parametrize("lens", [(1, 40), (20, 100), (20, 300), (200, 3000)])
def test_misaligned_runs_shift_kernel(sp, cuda, lens):
    """byte-granular hindexed displacements and lengths (word 1): runs of 32 B
    and more on average take k_runs_shift (16-B blocks of the written side
    assembled by funnel shifts), shorter ones the plain run kernel; pack and
    unpack of 3 objects vs the MPI typemap restatement, an unaligned packed
    position, and the bytes between runs untouched"""
    torch = cuda
    rng = np.random.default_rng(lens[1])
    n = 4000
    bls = rng.integers(lens[0], lens[1] + 1, n).tolist()
    gaps = rng.integers(0, 97, n).tolist()
    displs, at = [], 3
    for b, g in zip(bls, gaps):
        at += g
        displs.append(at)
        at += b
    perm = rng.permutation(n)
    bls = [bls[i] for i in perm]
    displs = [displs[i] for i in perm]
    c = sp.commit_type(sp.make_hindexed(bls, displs, sp.make_named(sp.NamedKind.Byte)))
    assert c.form == sp.CanonForm.Unsupported and not c.overlapping
    runs = list(zip(displs, bls))
    inc, pos = 3, 5
    span = (inc - 1) * c.extent + c.span
    host = rng.integers(0, 256, span, dtype=np.uint8)
    want = tm.gather(host, runs, inc, c.extent, c.size)
    dst = torch.full((pos + inc * c.size + 16,), 0xEE, dtype=torch.uint8, device="cuda")
    sp.pack(torch.from_numpy(host).cuda(), c, inc, dst, pos)
    li = sp.last_launch()
    shifted = c.size / n >= 32  # pack from a 32-B mean run, unpack from 512 B
    assert li.kernel == sp.Kernel.BlockList and li.word == (16 if shifted else 1), (li, c.size / n)
    got = dst.cpu().numpy()
    assert np.array_equal(got[pos:pos + inc * c.size], want)
    assert (got[:pos] == 0xEE).all() and (got[pos + inc * c.size:] == 0xEE).all()
    init = rng.integers(0, 256, span, dtype=np.uint8)
    out = torch.from_numpy(init.copy()).cuda()
    sp.unpack(dst, pos, c, inc, out)
    assert sp.last_launch().word == (16 if c.size / n >= 512 else 1)
    exp = tm.scatter(want, init.copy(), runs, inc, c.extent)
    assert np.array_equal(out.cpu().numpy(), exp)


@pytest.mark.gpu
def test_typed_copy_with_irregular_side(sp, cuda):
    """sp.copy (typed copy) with a block-list layout on one side and a dense
    run on the other: gather (irregular -> contiguous) and scatter
    (contiguous with a start offset -> irregular), 3 objects each; two
    irregular sides are refused"""
    torch = cuda
    rng = np.random.default_rng(8)
    D = sp.make_named(sp.NamedKind.Double)
    desc = ("indexed", [2, 1, 3, 2], [12, 0, 5, 20], ("named", 8))
    size, _, _, runs = tm.typemap(desc)
    irr = sp.commit_type(tm.build(sp, desc))
    assert irr.form == sp.CanonForm.Unsupported
    n = size // 8
    flat = sp.commit_type(sp.make_contiguous(n, D))
    host = rng.integers(0, 256, 3 * irr.extent + irr.span, dtype=np.uint8)
    want = tm.gather(host, runs, 3, irr.extent, size)
    src = torch.from_numpy(host).cuda()
    out = torch.zeros(3 * size, dtype=torch.uint8, device="cuda")
    sp.copy(src, irr, 3, out, flat, 3)
    assert np.array_equal(out.cpu().numpy(), want)
    # contiguous (offset 24, one object of 3*n doubles) -> irregular
    big = sp.commit_type(sp.make_hindexed([3 * n], [24], D))
    src2 = torch.zeros(24 + 3 * size, dtype=torch.uint8, device="cuda")
    src2[24:] = out
    back = torch.full((host.size,), 0x5A, dtype=torch.uint8, device="cuda")
    sp.copy(src2, big, 1, back, irr, 3)
    exp = tm.scatter(want, np.full(host.size, 0x5A, np.uint8), runs, 3, irr.extent)
    assert np.array_equal(back.cpu().numpy(), exp)
    with pytest.raises(sp.Unsupported):
        sp.copy(src, irr, 1, back, irr, 1)


def test_typed_copy_irregular_validation(sp):
    """validation before any launch (runs on CPU too): two irregular sides
    are refused, and byte counts must agree"""
    import torch
    D = sp.make_named(sp.NamedKind.Double)
    irr = sp.commit_type(sp.make_indexed([2, 1], [3, 0], D))
    flat = sp.commit_type(sp.make_contiguous(3, D))
    buf = torch.zeros(256, dtype=torch.uint8)
    with pytest.raises(sp.Unsupported):
        sp.copy(buf, irr, 1, buf, irr, 1)
    with pytest.raises(sp.InvalidArgument):
        sp.copy(buf, irr, 2, buf, flat, 1)
