"""GPU parity of pack/unpack (sm_100a kernels via the C-ABI) against the C
oracle and the reference's golden digests. Bit-exact: this is byte movement.

Restates proj/tests/test_pack.cpp (KATs, round trips with sentinels, oracle
gather equivalence, W-invariance, multi-count placement, bounds, overlap,
empty and fallback forms) and acceptance.cpp criterion 4, then adds what a
GPU executor must additionally get right: every kernel variant, unaligned
buffer addresses and positions, pinned and pageable host buffers, 64-bit
indexing, and the BASELINE configurations at full size.
"""
import hashlib
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def dev(torch, host):
    return torch.from_numpy(np.ascontiguousarray(host)).cuda()


def ramp(n):
    return (np.arange(n) & 0xFF).astype(np.uint8)


# ------------------------------------------------------------ KATs
def test_kat_vector_canonical_order(sp, cuda):
    """test_pack.cpp:44-58"""
    torch = cuda
    ct = sp.commit_type(sp.make_vector(3, 4, 8, sp.make_named(sp.NamedKind.Float)))
    src = dev(torch, ramp(96))
    dst = torch.zeros(48, dtype=torch.uint8, device="cuda")
    assert sp.pack(src, ct, 1, dst, 0) == 48
    want = np.concatenate([np.arange(b, b + 16) for b in (0, 32, 64)]).astype(np.uint8)
    assert np.array_equal(dst.cpu().numpy(), want)


def test_kat_single_byte_identity(sp, cuda):
    torch = cuda
    ct = sp.commit_type(sp.make_named(sp.NamedKind.Byte))
    src = torch.tensor([0xAB], dtype=torch.uint8, device="cuda")
    dst = torch.zeros(1, dtype=torch.uint8, device="cuda")
    assert sp.pack(src, ct, 1, dst, 0) == 1
    assert dst.item() == 0xAB


def test_kat_multiple_objects_one_extent_apart(sp, cuda):
    """test_pack.cpp:68-83"""
    torch = cuda
    ct = sp.commit_type(sp.make_vector(3, 4, 8, sp.make_named(sp.NamedKind.Float)))
    assert ct.extent == 80
    src = dev(torch, ramp(160))
    dst = torch.zeros(96, dtype=torch.uint8, device="cuda")
    assert sp.pack(src, ct, 2, dst, 0) == 96
    got = dst.cpu().numpy()
    for j in range(2):
        for i in range(3):
            for k in range(16):
                assert got[j * 48 + i * 16 + k] == (j * 80 + i * 32 + k) & 0xFF


def test_kat_interleaved_hvector(sp, cuda):
    """test_pack.cpp:185-198: visiting order is not address order"""
    torch = cuda
    b = sp.make_named(sp.NamedKind.Byte)
    ct = sp.commit_type(sp.make_hvector(2, 1, 10, sp.make_vector(3, 2, 8, b)))
    dst = torch.zeros(12, dtype=torch.uint8, device="cuda")
    sp.pack(dev(torch, ramp(28)), ct, 1, dst, 0)
    assert dst.cpu().tolist() == [0, 1, 8, 9, 16, 17, 10, 11, 18, 19, 26, 27]


def test_kat_four_dim(sp, cuda):
    """test_pack.cpp:200-239"""
    torch = cuda
    b = sp.make_named(sp.NamedKind.Byte)
    ct = sp.commit_type(sp.make_hvector(2, 1, 1000, sp.make_hvector(
        2, 1, 100, sp.make_hvector(2, 1, 10, sp.make_contiguous(2, b)))))
    host = np.random.default_rng(55).integers(0, 256, 1112, dtype=np.uint8)
    dst = torch.zeros(16, dtype=torch.uint8, device="cuda")
    sp.pack(dev(torch, host), ct, 1, dst, 0)
    want = [host[i3 * 1000 + i2 * 100 + i1 * 10 + k]
            for i3 in range(2) for i2 in range(2) for i1 in range(2) for k in range(2)]
    assert dst.cpu().tolist() == list(want)
    back = torch.full((1112,), 0x11, dtype=torch.uint8, device="cuda")
    sp.unpack(dst, 0, ct, 1, back)
    bk = back.cpu().numpy()
    for i3 in range(2):
        for i2 in range(2):
            for i1 in range(2):
                for k in range(2):
                    off = i3 * 1000 + i2 * 100 + i1 * 10 + k
                    assert bk[off] == host[off]


def test_kat_overlapping_pack_then_refuse_unpack(sp, cuda):
    """test_pack.cpp:241-261"""
    torch = cuda
    b = sp.make_named(sp.NamedKind.Byte)
    ct = sp.commit_type(sp.make_hvector(3, 1, 2, sp.make_contiguous(4, b)))
    assert ct.overlapping and ct.form == sp.CanonForm.Strided
    dst = torch.zeros(12, dtype=torch.uint8, device="cuda")
    sp.pack(dev(torch, ramp(8)), ct, 1, dst, 0)
    assert dst.cpu().tolist() == [0, 1, 2, 3, 2, 3, 4, 5, 4, 5, 6, 7]
    with pytest.raises(sp.OverlappingLayout):
        sp.unpack(dst, 0, ct, 1, torch.zeros(8, dtype=torch.uint8, device="cuda"))


def test_kat_empty_noop(sp, cuda):
    """test_pack.cpp:263-270"""
    torch = cuda
    ct = sp.commit_type(sp.make_vector(0, 4, 8, sp.make_named(sp.NamedKind.Float)))
    src = torch.ones(16, dtype=torch.uint8, device="cuda")
    dst = torch.full((16,), 2, dtype=torch.uint8, device="cuda")
    before = sp.kernel_launch_count()
    assert sp.pack(src, ct, 3, dst, 5) == 5
    assert sp.kernel_launch_count() == before
    assert dst.cpu().tolist() == [2] * 16


def test_kat_bounds(sp, cuda):
    """test_pack.cpp:272-289"""
    torch = cuda
    ct = sp.commit_type(sp.make_vector(3, 4, 8, sp.make_named(sp.NamedKind.Float)))
    z = lambda n: torch.zeros(n, dtype=torch.uint8, device="cuda")
    src = dev(torch, ramp(96))
    with pytest.raises(sp.BufferTooSmall):
        sp.pack(src, ct, 1, z(47), 0)
    with pytest.raises(sp.BufferTooSmall):
        sp.pack(z(79), ct, 1, z(48), 0)
    with pytest.raises(sp.InvalidArgument):
        sp.pack(src, ct, 0, z(48), 0)
    with pytest.raises(sp.BufferTooSmall):
        sp.unpack(z(48), 0, ct, 1, z(79))
    with pytest.raises(sp.BufferTooSmall):
        sp.unpack(z(47), 0, ct, 1, z(80))


def test_kat_unsupported_fallback(sp, cuda):
    """test_pack.cpp:291-303: definition-order gather on the device"""
    torch = cuda
    ct = sp.commit_type(sp.make_vector(2, 1, 0, sp.make_named(sp.NamedKind.Byte)))
    assert ct.form == sp.CanonForm.Unsupported
    src = torch.tensor([0x42], dtype=torch.uint8, device="cuda")
    dst = torch.zeros(2, dtype=torch.uint8, device="cuda")
    assert sp.pack(src, ct, 1, dst, 0) == 2
    assert sp.last_launch().kernel == sp.Kernel.BlockList
    assert dst.cpu().tolist() == [0x42, 0x42]
    with pytest.raises(sp.Unsupported):
        sp.pack(src, ct, 1, dst, 0, allow_fallback=False)
    with pytest.raises(sp.OverlappingLayout):
        sp.unpack(dst, 0, ct, 1, torch.zeros(1, dtype=torch.uint8, device="cuda"))


# ------------------------------------------------------------ golden digests
def test_reference_golden_digests(sp, cuda, pack_digests):
    """packed/unpacked bytes hash-equal to the REFERENCE's own outputs"""
    torch = cuda
    for row in pack_digests:
        ct = sp.commit_type(sp.from_program(row["prog"]))
        rng = np.random.default_rng(row["seed"])
        src = rng.integers(0, 256, (row["incount"] - 1) * ct.extent + ct.span, dtype=np.uint8)
        dst = torch.zeros(row["position"] + row["incount"] * ct.size, dtype=torch.uint8, device="cuda")
        sp.pack(dev(torch, src), ct, row["incount"], dst, row["position"])
        got = dst.cpu().numpy()
        assert _sha(got[row["position"]:]) == row["packed"], row["prog"]
        if "unpacked" in row:
            back = torch.full((len(src),), 0xCD, dtype=torch.uint8, device="cuda")
            sp.unpack(dst, row["position"], ct, row["incount"], back)
            assert _sha(back.cpu().numpy()) == row["unpacked"], row["prog"]


# ------------------------------------------------------------ randomized parity
KERNELS = ["auto", "words", "words_w1", "blocklist", "words64", "shift", "dma"]


def _opts(sp, ct, which):
    if which == "shift":
        return dict(kernel=sp.Kernel.Shift)
    if which == "words":
        return dict(kernel=sp.Kernel.Words)
    if which == "words_w1":
        return dict(kernel=sp.Kernel.Words, force_word=1)
    if which == "blocklist":
        return dict(kernel=sp.Kernel.BlockList)
    if which == "words64":
        return dict(kernel=sp.Kernel.Words64)
    if which == "dma":
        return dict(kernel=sp.Kernel.DMA)
    return {}


@pytest.mark.parametrize("which", KERNELS)
def test_corpus_parity_all_kernels(sp, orc, cuda, corpus, which):
    """pack == oracle gather and unpack round trip with sentinels, over the
    reference-generated corpus (acceptance.cpp:165-214, test_pack.cpp:99-183),
    for every kernel variant, with unaligned bases and positions."""
    torch = cuda
    rng = np.random.default_rng(KERNELS.index(which) + 7)
    checked = 0
    for e in corpus:
        r = e["ref"]
        if r["status"] or r["size"] == 0 or r["size"] > (1 << 15):
            continue
        prog = e["prog"]
        ct = sp.commit_type(sp.from_program(prog))
        if which in ("words64", "dma") and ct.form != sp.CanonForm.Strided:
            continue
        if which == "shift" and (ct.form != sp.CanonForm.Strided or ct.canon.counts[0] < 16):
            continue
        inc = 1 + int(rng.integers(0, 3))
        pos = int(rng.integers(0, 19))
        sshift = int(rng.integers(0, 16))
        span = (inc - 1) * ct.extent + ct.span
        host = rng.integers(0, 256, span, dtype=np.uint8)
        want = np.zeros(pos + inc * ct.size, np.uint8)
        st, npos = orc.pack(prog, host, inc, want, pos)
        assert st == 0
        sbuf = torch.zeros(span + 16, dtype=torch.uint8, device="cuda")
        sbuf[sshift:sshift + span] = dev(torch, host)
        src = sbuf[sshift:sshift + span]
        dbuf = torch.full((pos + inc * ct.size + 16,), 0xEE, dtype=torch.uint8, device="cuda")
        dshift = int(rng.integers(0, 16))
        dst = dbuf[dshift:dshift + pos + inc * ct.size]
        try:
            assert sp.pack(src, ct, inc, dst, pos, **_opts(sp, ct, which)) == npos
        except sp.Unsupported:  # the copy-engine path: overlapping rows or > 4096 pitched copies
            assert which == "dma"
            continue
        got = dbuf.cpu().numpy()
        assert np.array_equal(got[dshift + pos:dshift + pos + inc * ct.size], want[pos:]), prog
        assert (got[:dshift + pos] == 0xEE).all() and (got[dshift + pos + inc * ct.size:] == 0xEE).all()
        if not ct.overlapping:
            exp = np.full(span, 0x5A, np.uint8)
            assert orc.unpack(prog, want, pos, inc, exp)[0] == 0
            obuf = torch.full((span + 16,), 0x5A, dtype=torch.uint8, device="cuda")
            out = obuf[sshift:sshift + span]
            assert sp.unpack(dst, pos, ct, inc, out, **_opts(sp, ct, which)) == npos
            ob = obuf.cpu().numpy()
            assert np.array_equal(ob[sshift:sshift + span], exp), prog
            assert (ob[:sshift] == 0x5A).all() and (ob[sshift + span:] == 0x5A).all()
        checked += 1
    assert checked > (150 if which == "shift" else 400 if which == "dma" else 500)


@pytest.mark.parametrize("c0", [16, 17, 31, 33, 100, 255, 4099])
def test_shift_kernel_misaligned_rows(sp, orc, cuda, c0):
    """rows >= 16 B whose strided-side addresses are not word aligned (byte
    offsets into a subarray) run the funnel-shift kernel: exact for every
    strided / packed misalignment pair, sentinels intact on both sides"""
    torch = cuda
    rows = 37
    pitch = c0 + 5
    prog = [3, rows, 1, pitch, 1, c0, 0, 0]  # hvector(rows,1,pitch,contiguous(c0,BYTE))
    ct = sp.commit_type(sp.from_program(prog))
    rng = np.random.default_rng(c0)
    host = rng.integers(0, 256, ct.span, dtype=np.uint8)
    want = np.zeros(ct.size, np.uint8)
    assert orc.pack(prog, host, 1, want, 0)[0] == 0
    for sshift in (0, 1, 3, 8, 13):
        sbuf = torch.zeros(ct.span + 32, dtype=torch.uint8, device="cuda")
        sbuf[sshift:sshift + ct.span] = dev(torch, host)
        for dshift in (0, 5, 15):
            dbuf = torch.full((ct.size + 32,), 0xEE, dtype=torch.uint8, device="cuda")
            sp.pack(sbuf[sshift:sshift + ct.span], ct, 1, dbuf[dshift:dshift + ct.size], 0)
            li = sp.last_launch()
            assert li.kernel == sp.Kernel.Shift, li
            got = dbuf.cpu().numpy()
            assert np.array_equal(got[dshift:dshift + ct.size], want), (sshift, dshift)
            assert (got[:dshift] == 0xEE).all() and (got[dshift + ct.size:] == 0xEE).all()
            obuf = torch.full((ct.span + 32,), 0x5A, dtype=torch.uint8, device="cuda")
            sp.unpack(dbuf[dshift:dshift + ct.size], 0, ct, 1, obuf[sshift:sshift + ct.span],
                      kernel=sp.Kernel.Shift)
            assert sp.last_launch().kernel == sp.Kernel.Shift
            exp = np.full(ct.span, 0x5A, np.uint8)
            assert orc.unpack(prog, want, 0, 1, exp)[0] == 0
            ob = obuf.cpu().numpy()
            assert np.array_equal(ob[sshift:sshift + ct.span], exp), (sshift, dshift)
            assert (ob[:sshift] == 0x5A).all() and (ob[sshift + ct.span:] == 0x5A).all()
            # automatic choice: shift for unpack of long misaligned rows only
            obuf.fill_(0x5A)
            sp.unpack(dbuf[dshift:dshift + ct.size], 0, ct, 1, obuf[sshift:sshift + ct.span])
            auto = sp.last_launch().kernel
            assert auto == (sp.Kernel.Shift if c0 >= 128 else sp.Kernel.Words), (c0, auto)
            assert np.array_equal(obuf.cpu().numpy()[sshift:sshift + ct.span], exp)


def test_smallrow_kernel_selected_and_exact(sp, orc, cuda):
    """rows of 1/2/4/8 bytes go through the 16-byte assembling kernel, with
    head/tail chunks at every packed alignment"""
    torch = cuda
    for c0 in (1, 2, 4, 8):
        for rows in (1, 3, 17, 64, 1000):
            prog = [3, rows, 1, 40, 1, c0, 0, 0]  # hvector(rows,1,40,contiguous(c0,BYTE))
            ct = sp.commit_type(sp.from_program(prog))
            host = np.random.default_rng(rows * c0).integers(0, 256, ct.span, dtype=np.uint8)
            for pos in range(0, 32, c0):
                want = np.zeros(pos + ct.size, np.uint8)
                orc.pack(prog, host, 1, want, pos)
                dst = torch.zeros(pos + ct.size, dtype=torch.uint8, device="cuda")
                sp.pack(dev(torch, host), ct, 1, dst, pos)
                li = sp.last_launch()
                assert li.kernel == sp.Kernel.SmallRow, (c0, rows, li)
                assert np.array_equal(dst.cpu().numpy(), want), (c0, rows, pos)
                back = torch.full((ct.span,), 0x77, dtype=torch.uint8, device="cuda")
                sp.unpack(dst, pos, ct, 1, back)
                exp = np.full(ct.span, 0x77, np.uint8)
                orc.unpack(prog, want, pos, 1, exp)
                assert np.array_equal(back.cpu().numpy(), exp), (c0, rows, pos)


def test_word_invariance(sp, orc, cuda, corpus):
    """test_plan.cpp:134-150: output independent of the word size"""
    torch = cuda
    n = 0
    for e in corpus[:600]:
        r = e["ref"]
        if r["status"] or r["form"] != 0 or r["size"] > (1 << 14):
            continue
        ct = sp.commit_type(sp.from_program(e["prog"]))
        host = np.random.default_rng(n).integers(0, 256, ct.span, dtype=np.uint8)
        src = dev(torch, host)
        outs = []
        for w in (0, 1):
            dst = torch.zeros(ct.size, dtype=torch.uint8, device="cuda")
            sp.pack(src, ct, 1, dst, 0, kernel=sp.Kernel.Words, force_word=w)
            outs.append(dst.cpu().numpy())
        assert np.array_equal(outs[0], outs[1])
        n += 1
    assert n > 100


# ------------------------------------------------------------ host memory
def test_pinned_host_oneshot_and_pageable_staged(sp, orc, cuda):
    torch = cuda
    prog = [2, 4096, 1, 64, 0, 3]  # cfg1 shape at 4096 blocks
    ct = sp.commit_type(sp.from_program(prog))
    host = np.random.default_rng(3).integers(0, 256, ct.span, dtype=np.uint8)
    want = np.zeros(ct.size, np.uint8)
    orc.pack(prog, host, 1, want, 0)
    d_src = dev(torch, host)
    # device -> pinned host: the kernel stores straight into mapped memory
    pinned = torch.zeros(ct.size, dtype=torch.uint8).pin_memory()
    sp.pack(d_src, ct, 1, pinned, 0, sync=True)
    assert not sp.last_launch().staged
    assert np.array_equal(pinned.numpy(), want)
    # pageable numpy source and destination are staged through the device
    out = np.zeros(ct.size, np.uint8)
    sp.pack(host, ct, 1, out, 0)
    assert sp.last_launch().staged
    assert np.array_equal(out, want)
    # unpack from pinned host into device, and into pageable host
    back = torch.full((ct.span,), 0xCD, dtype=torch.uint8, device="cuda")
    p_src = torch.from_numpy(want.copy()).pin_memory()
    sp.unpack(p_src, 0, ct, 1, back, sync=True)
    exp = np.full(ct.span, 0xCD, np.uint8)
    orc.unpack(prog, want, 0, 1, exp)
    assert np.array_equal(back.cpu().numpy(), exp)
    hb = np.full(ct.span, 0xCD, np.uint8)
    sp.unpack(want, 0, ct, 1, hb)
    assert np.array_equal(hb, exp)


@pytest.mark.parametrize("e0", [8, 64, 512])
def test_copy_engine_path_pinned_host(sp, orc, cuda, e0):
    """Kernel.DMA (the copy engines, PAPER.md:1164's future work): a cfg2
    subarray packed from device memory straight into pinned host memory and
    unpacked back from it, 2 objects, vs the oracle"""
    torch = cuda
    prog, _ = cfg2_prog(e0)
    prog = list(prog)
    ct = sp.commit_type(sp.from_program(prog))
    inc = 2
    g = torch.Generator(device="cuda").manual_seed(77 + e0)
    span = (inc - 1) * ct.extent + ct.span
    src = torch.randint(0, 256, (span,), dtype=torch.uint8, device="cuda", generator=g)
    want = np.zeros(inc * ct.size, np.uint8)
    assert orc.pack(prog, src.cpu().numpy(), inc, want, 0)[0] == 0
    pinned = torch.zeros(inc * ct.size, dtype=torch.uint8).pin_memory()
    before = sp.kernel_launch_count()
    sp.pack(src, ct, inc, pinned, 0, kernel=sp.Kernel.DMA, sync=True)
    li = sp.last_launch()
    assert li.kernel == sp.Kernel.DMA and not li.staged and sp.kernel_launch_count() == before  # no SM kernel
    assert np.array_equal(pinned.numpy(), want)
    out = torch.randint(0, 256, (span,), dtype=torch.uint8, device="cuda", generator=g)
    exp = out.cpu().numpy()
    assert orc.unpack(prog, want, 0, inc, exp)[0] == 0
    sp.unpack(pinned, 0, ct, inc, out, kernel=sp.Kernel.DMA, sync=True)
    assert torch.equal(out, torch.from_numpy(exp).cuda())


def test_pinned_message_pipelined_dma(sp, orc, cuda):
    """a pinned-host packed message of many objects moves by chunked DMA
    (H2D of chunk k+1 overlapping the unpack of chunk k, D2H of chunk k the
    pack of chunk k+1, on a copy lane beside the caller's stream): bytes
    equal the oracle's at a nonzero position, and the call is complete on
    the caller's stream"""
    torch = cuda
    prog = [4, 3, 0, 256, 64, 32, 64, 32, 16, 8, 4, 2, 0, 0]  # 32 KiB objects, 512 KiB extent
    ct = sp.commit_type(sp.from_program(prog))
    n, pos = 300, 48  # 9.4 MiB packed: two 8 MiB chunks of whole objects
    span = (n - 1) * ct.extent + ct.span
    rng = np.random.default_rng(77)
    host = rng.integers(0, 256, span, dtype=np.uint8)
    want = np.zeros(pos + n * ct.size, np.uint8)
    assert orc.pack(prog, host, n, want, pos)[0] == 0
    s = torch.cuda.Stream()
    msg = torch.zeros(pos + n * ct.size, dtype=torch.uint8).pin_memory()
    src = dev(torch, host)
    torch.cuda.synchronize()
    assert sp.pack(src, ct, n, msg, pos, stream=s) == pos + n * ct.size
    li = sp.last_launch()
    s.synchronize()  # the caller's stream alone covers the whole call
    assert li.staged and li.launches == 2
    assert np.array_equal(msg.numpy(), want)
    init = rng.integers(0, 256, span, dtype=np.uint8)
    out = dev(torch, init)
    inmsg = torch.from_numpy(want.copy()).pin_memory()
    torch.cuda.synchronize()
    sp.unpack(inmsg, pos, ct, n, out, stream=s)
    s.synchronize()
    assert sp.last_launch().launches == 2
    exp = init.copy()
    assert orc.unpack(prog, want, pos, n, exp)[0] == 0
    assert np.array_equal(out.cpu().numpy(), exp)


# ------------------------------------------------------------ BASELINE configs
def cfg2_prog(e0):
    e2 = 2 ** math.ceil(math.log2((1 << 20) // e0) / 2)
    e1 = (1 << 20) // (e0 * e2)
    return [4, 3, 0, 1024, 1024, 1024, e0, e1, e2, 0, 0, 0, 0, 0], (e0, e1, e2)


def test_cfg1_full_size(sp, orc, cuda):
    """vector(131072,1,64,DOUBLE): 1 MiB of 8 B blocks at 512 B pitch"""
    torch = cuda
    prog = [2, 131072, 1, 64, 0, 3]
    ct = sp.commit_type(sp.from_program(prog))
    host = np.random.default_rng(1).integers(0, 256, ct.span, dtype=np.uint8)
    want = np.zeros(ct.size, np.uint8)
    orc.pack(prog, host, 1, want, 0)
    dst = torch.zeros(ct.size, dtype=torch.uint8, device="cuda")
    sp.pack(dev(torch, host), ct, 1, dst, 0)
    assert np.array_equal(dst.cpu().numpy(), want)
    back = torch.full((ct.span,), 0xCD, dtype=torch.uint8, device="cuda")
    sp.unpack(dst, 0, ct, 1, back)
    exp = np.full(ct.span, 0xCD, np.uint8)
    orc.unpack(prog, want, 0, 1, exp)
    assert np.array_equal(back.cpu().numpy(), exp)


# ------------------------------------------------------------ TMA path
def test_tma_path_parity(sp, orc, cuda, corpus):
    """the TMA-tiled kernels (tensor-map box staged through shared memory)
    produce the oracle's bytes wherever they apply; rows clipped at tile
    edges are never written on unpack"""
    torch = cuda
    rng = np.random.default_rng(404)
    n = 0
    for e in corpus:
        r = e["ref"]
        if r["status"] or r["form"] != 0 or r["size"] > (1 << 15) or r["overlapping"]:
            continue
        prog = e["prog"]
        ct = sp.commit_type(sp.from_program(prog))
        inc = 1 + int(rng.integers(0, 2))
        span = (inc - 1) * ct.extent + ct.span
        host = rng.integers(0, 256, span, dtype=np.uint8)
        src = dev(torch, host)
        dst = torch.zeros(inc * ct.size, dtype=torch.uint8, device="cuda")
        try:
            sp.pack(src, ct, inc, dst, 0, kernel=sp.Kernel.TMA)
        except sp.InvalidArgument:
            continue
        assert sp.last_launch().kernel == sp.Kernel.TMA
        want = np.zeros(inc * ct.size, np.uint8)
        orc.pack(prog, host, inc, want, 0)
        assert np.array_equal(dst.cpu().numpy(), want), prog
        back = torch.full((span,), 0x6B, dtype=torch.uint8, device="cuda")
        sp.unpack(dst, 0, ct, inc, back, kernel=sp.Kernel.TMA)
        exp = np.full(span, 0x6B, np.uint8)
        orc.unpack(prog, want, 0, inc, exp)
        assert np.array_equal(back.cpu().numpy(), exp), prog
        n += 1
    # hand-built shapes that exercise partial tiles, 4 row dims and counts
    shapes = [[3, 300, 1, 64, 1, 48, 0, 0],
              [3, 3, 1, 16384, 3, 257, 1, 32, 1, 16, 0, 0],
              [3, 2, 1, 1 << 16, 3, 3, 1, 8192, 3, 5, 1, 512, 1, 256, 0, 0]]
    for prog in shapes:
        ct = sp.commit_type(sp.from_program(prog))
        for inc in (1, 3):
            span = (inc - 1) * ct.extent + ct.span
            host = rng.integers(0, 256, span, dtype=np.uint8)
            dst = torch.zeros(inc * ct.size, dtype=torch.uint8, device="cuda")
            sp.pack(dev(torch, host), ct, inc, dst, 0, kernel=sp.Kernel.TMA)
            assert sp.last_launch().kernel == sp.Kernel.TMA
            want = np.zeros(inc * ct.size, np.uint8)
            assert orc.pack(prog, host, inc, want, 0)[0] == 0
            assert np.array_equal(dst.cpu().numpy(), want), prog
            init = rng.integers(0, 256, span, dtype=np.uint8)
            back = dev(torch, init)
            sp.unpack(dst, 0, ct, inc, back, kernel=sp.Kernel.TMA)
            exp = init.copy()
            assert orc.unpack(prog, want, 0, inc, exp)[0] == 0
            assert np.array_equal(back.cpu().numpy(), exp), prog
            n += 1
    assert n > 20


@pytest.mark.parametrize("kernel", ["auto", "words", "tma", "dma"])
@pytest.mark.parametrize("e0", [1, 2, 4, 8, 16, 32, 64, 128, 256, 512])
def test_cfg2_full_size_vs_oracle(sp, orc, cuda, e0, kernel):
    """cfg2 at full size, pack AND unpack byte-compared with the oracle over
    the whole 1 GiB allocation: the unpack target starts as random bytes
    (not a constant), so every byte outside the described ones must survive
    untouched. kernel = the automatic choice (TMA for unpack of rows >= 64 B
    at this size), the LDG/STG word kernel, and the TMA path forced (rows of
    16 B and up), and the copy engines (cudaMemcpy3DAsync, no kernel)."""
    torch = cuda
    if kernel == "tma" and e0 < 16:
        pytest.skip("the TMA path needs rows that are a multiple of 16 B")
    k = {"auto": sp.Kernel.Auto, "words": sp.Kernel.Words, "tma": sp.Kernel.TMA, "dma": sp.Kernel.DMA}[kernel]
    prog, _ = cfg2_prog(e0)
    ct = sp.commit_type(sp.from_program(prog))
    g = torch.Generator(device="cuda").manual_seed(1000 + e0)
    src = torch.randint(0, 256, (ct.span,), dtype=torch.uint8, device="cuda", generator=g)
    host = src.cpu().numpy()
    want = np.zeros(ct.size, np.uint8)
    assert orc.pack(prog, host, 1, want, 0)[0] == 0
    dst = torch.zeros(ct.size, dtype=torch.uint8, device="cuda")
    sp.pack(src, ct, 1, dst, 0, kernel=k)
    if kernel != "auto":
        assert sp.last_launch().kernel == k
    assert np.array_equal(dst.cpu().numpy(), want)
    # unpack the oracle's packed bytes over a random 1 GiB target
    out = torch.randint(0, 256, (ct.span,), dtype=torch.uint8, device="cuda", generator=g)
    exp = out.cpu().numpy()
    assert orc.unpack(prog, want, 0, 1, exp)[0] == 0
    sp.unpack(torch.from_numpy(want).cuda(), 0, ct, 1, out, kernel=k)
    if kernel != "auto":
        assert sp.last_launch().kernel == k
    del src
    assert torch.equal(out, torch.from_numpy(exp).cuda())


def test_cfg1_incount64_vs_oracle(sp, orc, cuda):
    """BASELINE config 1 at the throughput count: 64 vector objects one
    extent apart (a 4.3 GB span), pack and unpack byte-compared with the
    oracle over the whole span"""
    torch = cuda
    prog = [2, 131072, 1, 64, 0, 3]
    ct = sp.commit_type(sp.from_program(prog))
    n = 64
    span = (n - 1) * ct.extent + ct.span
    g = torch.Generator(device="cuda").manual_seed(64)
    src = torch.randint(0, 256, (span,), dtype=torch.uint8, device="cuda", generator=g)
    host = src.cpu().numpy()
    want = np.zeros(n * ct.size, np.uint8)
    assert orc.pack(prog, host, n, want, 0)[0] == 0
    dst = torch.zeros(n * ct.size, dtype=torch.uint8, device="cuda")
    sp.pack(src, ct, n, dst, 0)
    assert np.array_equal(dst.cpu().numpy(), want)
    del src
    out = torch.randint(0, 256, (span,), dtype=torch.uint8, device="cuda", generator=g)
    exp = out.cpu().numpy()
    assert orc.unpack(prog, want, 0, n, exp)[0] == 0
    sp.unpack(dst, 0, ct, n, out)
    assert torch.equal(out, torch.from_numpy(exp).cuda())


# ------------------------------------------------------------ config 3
def test_cfg3_constructions_identical(sp, cuda):
    """BASELINE config 3: the cfg2 object (E0=32) built five ways reaches one
    StridedBlock and one plan, and packs to identical bytes"""
    torch = cuda
    e0, e1, e2 = 32, 128, 256
    b = sp.make_named(sp.NamedKind.Byte)
    ways = [
        sp.make_subarray(3, [1024] * 3, [e0, e1, e2], [0, 0, 0], b),
        sp.make_hvector(e2, 1, 1 << 20, sp.make_vector(e1, e0, 1024, b)),
        sp.make_hvector(e2, 1, 1 << 20, sp.make_vector(e1, 1, 1024 // e0, sp.make_hvector(e0, 1, 1, b))),
        sp.make_hvector(e2, 1, 1 << 20, sp.make_hvector(e1, 1, 1024, sp.make_contiguous(e0, b))),
        sp.make_subarray(1, [1024], [e2], [0], sp.make_subarray(2, [1024, 1024], [e0, e1], [0, 0], b)),
    ]
    cts = [sp.commit_type(w) for w in ways]
    assert len({(c.canon, c.plan) for c in cts}) == 1
    assert cts[0].canon == sp.StridedBlock(0, (e0, e1, e2), (1, 1024, 1 << 20))
    span = max(c.span for c in cts)
    g = torch.Generator(device="cuda").manual_seed(3)
    src = torch.randint(0, 256, (span,), dtype=torch.uint8, device="cuda", generator=g)
    outs = []
    for c in cts:
        o = torch.empty(c.size, dtype=torch.uint8, device="cuda")
        sp.pack(src, c, 1, o, 0)
        outs.append(o)
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


@pytest.mark.gpu
@pytest.mark.parametrize("e0", [1, 2, 4, 8, 16, 64, 128, 256, 512])
def test_cfg3_constructions_identical_every_e0(sp, cuda, e0):
    """BASELINE config 3 across the whole E0 sweep of config 2 (E0 = 32 is
    the test above): the five constructions reach one StridedBlock and plan,
    pack to identical bytes, and unpack those bytes to identical buffers
    (each through the kernel the engine picks for that E0)"""
    torch = cuda
    e2 = 2 ** math.ceil(math.log2((1 << 20) // e0) / 2)
    e1 = (1 << 20) // (e0 * e2)
    b = sp.make_named(sp.NamedKind.Byte)
    ways = [
        sp.make_subarray(3, [1024] * 3, [e0, e1, e2], [0, 0, 0], b),
        sp.make_hvector(e2, 1, 1 << 20, sp.make_vector(e1, e0, 1024, b)),
        sp.make_hvector(e2, 1, 1 << 20, sp.make_vector(e1, 1, 1024 // e0, sp.make_hvector(e0, 1, 1, b))),
        sp.make_hvector(e2, 1, 1 << 20, sp.make_hvector(e1, 1, 1024, sp.make_contiguous(e0, b))),
        sp.make_subarray(1, [1024], [e2], [0], sp.make_subarray(2, [1024, 1024], [e0, e1], [0, 0], b)),
    ]
    cts = [sp.commit_type(w) for w in ways]
    assert len({(c.canon, c.plan) for c in cts}) == 1, [c.canon for c in cts]
    span = max(c.span for c in cts)
    g = torch.Generator(device="cuda").manual_seed(300 + e0)
    src = torch.randint(0, 256, (span,), dtype=torch.uint8, device="cuda", generator=g)
    outs = []
    for c in cts:
        o = torch.empty(c.size, dtype=torch.uint8, device="cuda")
        sp.pack(src, c, 1, o, 0)
        outs.append(o)
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    # unpack: the described bytes land, everything else keeps its sentinel
    first = None
    for c in cts:
        dst = torch.full((span,), 0xA5, dtype=torch.uint8, device="cuda")
        sp.unpack(outs[0], 0, c, 1, dst)
        if first is None:
            first = dst
            assert int((dst != 0xA5).sum()) <= c.size
            assert torch.equal(dst.view(-1)[: e0], src[: e0])
        else:
            assert torch.equal(dst, first)
            del dst
    del src, first


def test_concurrent_host_threads_share_committed_types(sp, orc, cuda):
    """The reference's threading contract (commit.hpp:81-84):
    committed types are shared read-only and pack/unpack may run from many
    threads at once given exclusive destinations. Here 8 host threads, each
    on its own CUDA stream, pack and unpack the same committed types (cfg1
    and cfg2 shapes, every small-row and word kernel, device and pageable
    host buffers) while other threads commit; every result is checked
    against the oracle."""
    import threading
    torch = cuda
    # cfg1 at 4096 blocks and cfg2-shaped subarrays (1024-B pitch, 64 KiB
    # planes) small enough for the oracle
    progs = [[2, 4096, 1, 64, 0, 3]] + [[4, 3, 0, 1024, 64, 16, e0, 32, 8, 1, 2, 3, 0, 0]
                                        for e0 in (1, 4, 16, 64)]
    cts = [sp.commit_type(sp.from_program(p)) for p in progs]
    rng = np.random.default_rng(21)
    hosts = [rng.integers(0, 256, c.span, dtype=np.uint8) for c in cts]
    wants = []
    for p, c, h in zip(progs, cts, hosts):
        w = np.zeros(c.size, np.uint8)
        assert orc.pack(p, h, 1, w, 0)[0] == 0
        wants.append(w)
    srcs = [dev(torch, h) for h in hosts]  # shared, read-only
    errors = []

    def work(t):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            for it in range(6):
                k = (t + it) % len(cts)
                c = cts[k]
                out = torch.empty(c.size, dtype=torch.uint8, device="cuda")
                sp.pack(srcs[k], c, 1, out, 0, stream=s)
                back = torch.zeros(c.span, dtype=torch.uint8, device="cuda")
                sp.unpack(out, 0, c, 1, back, stream=s)
                s.synchronize()
                if not np.array_equal(out.cpu().numpy(), wants[k]):
                    errors.append((t, it, "pack"))
                exp = torch.from_numpy(hosts[k]).cuda()
                mask = torch.zeros(c.span, dtype=torch.uint8)
                mask_np = mask.numpy()
                orc.unpack(progs[k], np.ones(c.size, np.uint8), 0, 1, mask_np)
                m = torch.from_numpy(mask_np).cuda().bool()
                if not torch.equal(back[m], exp[m]) or back[~m].any():
                    errors.append((t, it, "unpack"))
                if t % 4 == 3:  # pageable host destination: staged path
                    hout = np.zeros(c.size, np.uint8)
                    sp.pack(hosts[k], c, 1, hout, 0)
                    if not np.array_equal(hout, wants[k]):
                        errors.append((t, it, "staged"))
                if t % 4 == 2:  # commits racing the packs
                    sp.commit_type(sp.make_vector(1 + it, 1 + t, 8 + t, sp.make_named(sp.NamedKind.Double)))
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append((t, repr(e)))

    ths = [threading.Thread(target=work, args=(t,)) for t in range(8)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert not errors, errors[:5]


@pytest.mark.gpu
def test_pack_unpack_replay_from_cuda_graph(sp, orc, cuda):
    """CUDA graphs instead of a tracing compiler: sp_pack / sp_unpack of
    device buffers enqueue only kernels, so an application can capture them
    (here a cfg2-shaped subarray and the cfg1 vector, pack then unpack) into
    one graph and replay it; every replay with fresh source bytes matches
    the oracle, and bytes outside the layout keep the sentinel"""
    torch = cuda
    progs = [[4, 3, 0, 1024, 64, 16, 16, 32, 8, 1, 2, 3, 0, 0], [2, 4096, 1, 64, 0, 3]]
    cts = [sp.commit_type(sp.from_program(p)) for p in progs]
    srcs = [torch.empty(c.span, dtype=torch.uint8, device="cuda") for c in cts]
    packs = [torch.empty(c.size, dtype=torch.uint8, device="cuda") for c in cts]
    backs = [torch.empty(c.span, dtype=torch.uint8, device="cuda") for c in cts]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):  # first launches (module load, occupancy queries) outside the capture
        for c, a, p, b in zip(cts, srcs, packs, backs):
            sp.pack(a, c, 1, p, 0)
            sp.unpack(p, 0, c, 1, b)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for c, a, p, b in zip(cts, srcs, packs, backs):
            sp.pack(a, c, 1, p, 0)
            sp.unpack(p, 0, c, 1, b)
    rng = np.random.default_rng(77)
    for rep in range(3):
        hosts = [rng.integers(0, 256, c.span, dtype=np.uint8) for c in cts]
        for a, b, h in zip(srcs, backs, hosts):
            a.copy_(torch.from_numpy(h))
            b.fill_(0xC3)
        torch.cuda.synchronize()
        before = sp.kernel_launch_count()
        g.replay()
        torch.cuda.synchronize()
        assert sp.kernel_launch_count() == before  # replayed by the driver, not re-enqueued by the engine
        for prog, c, p, b, h in zip(progs, cts, packs, backs, hosts):
            want = np.zeros(c.size, np.uint8)
            assert orc.pack(prog, h, 1, want, 0)[0] == 0
            assert np.array_equal(p.cpu().numpy(), want), (rep, prog)
            exp = np.full(c.span, 0xC3, np.uint8)
            assert orc.unpack(prog, want, 0, 1, exp)[0] == 0
            assert np.array_equal(b.cpu().numpy(), exp), (rep, prog)
