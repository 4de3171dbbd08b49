"""Host-side commit pipeline of the product (libstridepack_b200.so) against
the reference's golden results and known-answer tests. CPU only: commit,
canonicalisation, plan and overlap are host logic.

KATs restate the reference's own tests: proj/tests/test_typemodel.cpp,
test_canon.cpp, test_plan.cpp, test_pack.cpp and acceptance.cpp criterion 1.
"""
import threading

import pytest


def record(sp, prog):
    try:
        ct = sp.commit_type(sp.from_program(prog))
    except sp.InvalidArgument:
        return {"status": 1}
    except sp.UnsupportedOrder:
        return {"status": 2}
    rec = {"status": 0, "form": int(ct.form), "size": ct.size, "extent": ct.extent,
           "span": ct.span, "overlapping": int(ct.overlapping),
           "n_fallback_runs": ct.n_fallback_runs}
    if ct.form == sp.CanonForm.Strided:
        rec.update(start=ct.canon.start, counts=list(ct.canon.counts),
                   strides=list(ct.canon.strides), word=ct.plan.word,
                   block=list(ct.plan.block_dims), grid=list(ct.plan.grid_dims),
                   strategy=int(ct.plan.count_strategy), rounds=ct.simplify_rounds)
    return rec


def test_commit_matches_reference_on_golden_corpus(sp, corpus):
    bad = [(e["set"], e["i"]) for e in corpus if record(sp, e["prog"]) != e["ref"]]
    assert not bad, bad[:10]


@pytest.mark.parametrize("seed,mode", [(11, 2), (12, 0), (13, 1), (14, 2)])
def test_commit_matches_live_reference(sp, ref, seed, mode):
    for prog in ref.corpus(seed, 500, mode):
        want = ref.commit(prog)
        got = record(sp, prog)
        assert got["status"] == want.status, prog
        if want.status:
            continue
        assert (got["form"], got["size"], got["extent"], got["span"], bool(got["overlapping"])) == \
            (want.form, want.size, want.extent, want.span, want.overlapping), prog
        if want.form == 0:
            assert (got["start"], got["counts"], got["strides"], got["word"]) == \
                (want.start, want.counts, want.strides, want.word), prog


B = None


def byte(sp):
    return sp.make_named(sp.NamedKind.Byte)


def flt(sp):
    return sp.make_named(sp.NamedKind.Float)


def canon_of(sp, d):
    ct = sp.commit_type(d)
    return (ct.canon.start, ct.canon.counts, ct.canon.strides) if ct.canon else None


def test_construction_zoo_acceptance_c1(sp):
    """acceptance.cpp:71-132: 20 constructions of a row/plane/cuboid."""
    b, f = byte(sp), flt(sp)
    rows = [sp.make_contiguous(100, f), sp.make_contiguous(400, b), sp.make_vector(1, 100, 1, f),
            sp.make_vector(100, 4, 4, b), sp.make_hvector(400, 1, 1, b),
            sp.make_subarray(1, [256], [400], [0], b), sp.make_subarray(1, [1024], [400], [0], b)]
    sub_row = rows[5]
    planes = [sp.make_vector(13, 100, 64, f), sp.make_vector(13, 400, 256, b),
              sp.make_subarray(2, [256, 512], [400, 13], [0, 0], b),
              sp.make_hvector(13, 1, 256, rows[0]), sp.make_hvector(13, 1, 256, rows[3]),
              sp.make_hvector(13, 1, 256, sub_row), sp.make_vector(13, 1, 1, sub_row),
              sp.make_subarray(1, [512], [13], [0], sub_row)]
    cuboids = [sp.make_subarray(3, [256, 512, 1024], [400, 13, 47], [0, 0, 0], b),
               sp.make_hvector(47, 1, 131072, planes[0]),
               sp.make_hvector(47, 1, 131072, sp.make_hvector(13, 1, 256, sp.make_contiguous(400, b))),
               sp.make_hvector(47, 1, 131072, planes[2]),
               sp.make_hvector(13, 1, 256, sp.make_hvector(47, 1, 131072, sp.make_contiguous(400, b)))]
    for r in rows:
        assert canon_of(sp, r) == (0, (400,), (1,))
    for p in planes:
        assert canon_of(sp, p) == (0, (400, 13), (1, 256))
    for c in cuboids:
        assert canon_of(sp, c) == (0, (400, 13, 47), (1, 256, 131072))


def test_typemodel_kats(sp):
    """test_typemodel.cpp:16-96"""
    b, f = byte(sp), flt(sp)
    assert sp.make_named(sp.NamedKind.Double).size() == 8
    assert sp.make_contiguous(100, f).size() == 400
    with pytest.raises(sp.InvalidArgument):
        sp.make_subarray(1, [8], [4], [6], b)
    with pytest.raises(sp.InvalidArgument):
        sp.make_subarray(2, [8], [4], [0], b)
    with pytest.raises(sp.UnsupportedOrder):
        sp.make_subarray(1, [8], [4], [0], b, sp.ArrayOrder.Fortran)
    with pytest.raises(sp.InvalidArgument):
        sp.make_contiguous(-1, b)
    with pytest.raises(sp.InvalidArgument):
        sp.make_vector(2, 1, -3, b)
    with pytest.raises(sp.InvalidArgument):
        sp.make_hvector(2, 1, -3, b)
    with pytest.raises(sp.InvalidArgument):
        sp.make_subarray(1, [0], [1], [0], b)
    empty = sp.make_vector(0, 4, 8, f)
    assert empty.size() == 0 and empty.extent() == 0
    sp.make_subarray(1, [256], [400], [0], b)  # oversized dim at offset 0 is legal
    assert sp.make_vector(3, 4, 8, f).size() == 48
    assert sp.make_vector(3, 4, 8, f).extent() == 80
    assert sp.make_subarray(3, [256, 512, 1024], [400, 13, 47], [0, 0, 0], b).size() == 244400
    assert sp.make_hvector(13, 1, 256, sp.make_contiguous(400, b)).extent() == 3472
    ct = sp.commit_type(f)
    assert ct.canon == sp.StridedBlock(0, (4,), (1,)) and ct.size == 4 and ct.extent == 4
    ce = sp.commit_type(empty)
    assert ce.form == sp.CanonForm.Empty and ce.size == 0 and ce.span == 0


def test_overlap_flagged_not_forbidden(sp):
    b = byte(sp)
    ct = sp.commit_type(sp.make_hvector(13, 1, 256, sp.make_contiguous(400, b)))
    assert ct.overlapping and ct.form == sp.CanonForm.Strided
    assert ct.canon == sp.StridedBlock(0, (400, 13), (1, 256))
    ct = sp.commit_type(sp.make_hvector(2, 1, 10, sp.make_vector(3, 2, 8, b)))
    assert not ct.overlapping  # interleaved but disjoint (test_pack.cpp:185-198)
    assert ct.canon == sp.StridedBlock(0, (2, 3, 2), (1, 8, 10))


def test_coincident_elements_are_unsupported(sp):
    """test_canon.cpp:177-189: commit never fails, it stores the marker."""
    ct = sp.commit_type(sp.make_vector(2, 1, 0, byte(sp)))
    assert ct.form == sp.CanonForm.Unsupported and ct.canon is None and ct.plan is None
    assert ct.overlapping and ct.n_fallback_runs == 2 and ct.size == 2 and ct.span == 1


def test_plan_kats(sp):
    """test_plan.cpp:43-78 expressed through committed definitions."""
    b = byte(sp)
    ct = sp.commit_type(sp.make_subarray(3, [256, 512, 1024], [400, 13, 47], [0, 0, 0], b))
    assert ct.plan == sp.PackPlan(16, (32, 16, 2), (1, 1, 24), sp.CountStrategy.Iterate)
    ct = sp.commit_type(sp.make_contiguous(4, b))
    assert ct.plan == sp.PackPlan(4, (1, 1, 1), (1, 1, 1), sp.CountStrategy.GridZ)
    ct = sp.commit_type(sp.make_hvector(1024, 1, 8192, sp.make_contiguous(512, b)))
    assert ct.plan == sp.PackPlan(16, (32, 32, 1), (1, 32, 1), sp.CountStrategy.GridZ)
    ct = sp.commit_type(sp.make_contiguous(1 << 16, b))
    assert ct.plan.word == 16 and ct.plan.block_dims[0] == 1024 and ct.plan.grid_dims[0] == 4
    ct = sp.commit_type(sp.make_subarray(3, [512, 512, 1024], [400, 13, 47], [2, 0, 0], b))
    assert ct.canon.start == 2 and ct.plan.word == 2
    assert sp.commit_type(sp.make_contiguous(3, b)).plan.word == 1
    assert sp.commit_type(sp.make_hvector(5, 1, 260, sp.make_contiguous(400, b))).plan.word == 4


def test_four_dim_iterate(sp):
    """test_pack.cpp:200-212"""
    b = byte(sp)
    d = sp.make_hvector(2, 1, 1000, sp.make_hvector(2, 1, 100, sp.make_hvector(2, 1, 10, sp.make_contiguous(2, b))))
    ct = sp.commit_type(d)
    assert ct.canon == sp.StridedBlock(0, (2, 2, 2, 2), (1, 10, 100, 1000))
    assert ct.plan.count_strategy == sp.CountStrategy.Iterate


def test_baseline_config_canon(sp):
    """cfg1 and the cfg2 sweep reach the stated forms."""
    d = sp.make_vector(131072, 1, 64, sp.make_named(sp.NamedKind.Double))
    ct = sp.commit_type(d)
    assert ct.canon == sp.StridedBlock(0, (8, 131072), (1, 512))
    assert ct.plan == sp.PackPlan(8, (1, 1024, 1), (1, 128, 1), sp.CountStrategy.GridZ)
    for e0, want in [(1, (1, 1048576)), (8, (8, 256, 512)), (32, (32, 128, 256)), (512, (512, 32, 64))]:
        import math
        e2 = 2 ** math.ceil(math.log2((1 << 20) // e0) / 2)
        e1 = (1 << 20) // (e0 * e2)
        ct = sp.commit_type(sp.make_subarray(3, [1024] * 3, [e0, e1, e2], [0, 0, 0], byte(sp)))
        assert ct.canon.counts == want, (e0, ct.canon)
        assert ct.size == 1 << 20 and ct.extent == 1 << 30
        assert not ct.overlapping


def test_commit_is_deterministic_and_idempotent(sp):
    d = sp.make_vector(5, 2, 3, sp.make_subarray(2, [8, 4], [4, 2], [1, 1], sp.make_named(sp.NamedKind.Int)))
    a = sp.commit_type(d)
    b = sp.commit_type(d)
    assert a.canon == b.canon and a.plan == b.plan and a.size == b.size


def test_concurrent_commits(sp):
    """test_typemodel.cpp:145-170"""
    out = [None] * 64
    b = byte(sp)

    def work(t):
        for i in range(16):
            d = sp.make_contiguous(t * 16 + i + 1, b)
            out[t * 16 + i] = (d, sp.commit_type(d).size)

    ths = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert sorted(s for _, s in out) == list(range(1, 65))
    assert len({d.handle for d, _ in out}) == 64


def test_invalid_handle(sp):
    from paper_2012_14363_b200 import _capi
    import ctypes as C
    v = C.c_int64()
    assert _capi.lib.sp_type_size(0, C.byref(v)) == 11
    assert _capi.lib.sp_type_commit(1 << 60) == 11


def test_exact_overlap_hard_cases(sp, orc):
    """Interleaved lattices where the nested-span shortcut is inconclusive:
    the exact search must agree with the oracle's block-list normalisation."""
    import itertools
    b = byte(sp)
    cases = 0
    for c0, s1, c1, s2, c2 in itertools.product([1, 2, 3, 5], [4, 6, 7], [2, 3, 5], [9, 10, 13, 15], [2, 3, 4]):
        prog = [3, c2, 1, s2, 3, c1, 1, s1, 1, c0, 0, 0]
        want = orc.commit(prog)
        got = sp.commit_type(sp.from_program(prog))
        assert got.overlapping == want.overlapping, prog
        cases += 1
    assert cases > 100


@pytest.mark.parametrize("seed", range(4))
def test_random_cuboids_reach_one_canonical_form(sp, seed):
    """north_star / SURVEY §8a T3-T5: a 3-D block built five ways (subarray,
    hvector of vector, nested hvectors of a contiguous row, a vector of that
    plane resized to the plane pitch, and hvector of a Double vector)
    commits to one StridedBlock. Random shapes; cfg3 (BASELINE config 3) is
    the fixed case.
    The reference's acceptance.cpp:71-132 zoo is the pattern followed."""
    import random
    rng = random.Random(1000 + seed)
    b = byte(sp)
    dbl = sp.make_named(sp.NamedKind.Double)
    for _ in range(50):
        e0 = 8 * rng.randint(1, 16)  # a multiple of 8 B so the Double form exists
        a0 = e0 + 8 * rng.randint(1, 8)  # a multiple of 8 as well
        e1, e2 = rng.randint(2, 9), rng.randint(2, 9)
        a1 = e1 + rng.randint(1, 4)
        a2 = e2 + rng.randint(0, 3)
        row = sp.make_contiguous(e0, b)
        plane = sp.make_hvector(e1, 1, a0, row)
        forms = [
            sp.make_subarray(3, [a0, a1, a2], [e0, e1, e2], [0, 0, 0], b),
            sp.make_hvector(e2, 1, a0 * a1, sp.make_vector(e1, e0, a0, b)),
            sp.make_hvector(e2, 1, a0 * a1, plane),
            sp.make_vector(e2, 1, 1, sp.make_resized(plane, 0, a0 * a1)),
            sp.make_hvector(e2, 1, a0 * a1, sp.make_vector(e1, e0 // 8, a0 // 8, dbl)),
        ]
        want = (0, (e0, e1, e2), (1, a0, a0 * a1))
        for i, d in enumerate(forms):
            ct = sp.commit_type(d)
            assert (ct.canon.start, ct.canon.counts, ct.canon.strides) == want, (i, e0, e1, e2, a0, a1, ct.canon)
            assert ct.size == e0 * e1 * e2 and not ct.overlapping
