"""The command-line front end and type-file language:
tools/stridepack against the reference's proj/tests/test_cli.cpp cases (same
inputs, same expected strings and exit codes), the type-file parser against
the reference-generated corpus (tests/golden/corpus.json: every definition
written out as a type file must commit to the reference's canonical form),
and `halo` output against the reference's own run_exchange reports
(tests/golden/halo_golden.json) formatted as cli.hpp:249-266 prints them.

canon / flatten / choose / parse errors run on CPU; pack / unpack / halo /
profile-gen execute on the B200 (-m gpu)."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "stridepack")
GOLD = os.path.join(ROOT, "tests", "golden")
PROFILE = os.path.join(GOLD, "default.profile")

CUBOID = ("# cuboid built as hvector of hvector of bytes\n"
          "type row = contiguous(400, byte)\n"
          "type plane = hvector(13, 1, 256, row)\n"
          "type cuboid = hvector(47, 1, 131072, plane)\n"
          "commit cuboid\n")
VEC = "type t = vector(3, 4, 8, float)\ncommit t\n"
OVERLAP = "type row = contiguous(400, byte)\ntype t = hvector(13, 1, 256, row)\ncommit t\n"


def run(*args):
    if not os.path.exists(CLI):
        pytest.fail(f"{CLI} not built (run __graft_entry__.build())")
    p = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=300)
    return p.returncode, p.stdout, p.stderr


@pytest.fixture
def tf(tmp_path):
    def write(name, content):
        p = tmp_path / name
        if isinstance(content, (bytes, bytearray)):
            p.write_bytes(bytes(content))
        else:
            p.write_text(content)
        return str(p)
    write.dir = tmp_path
    return write


def ramp(n):
    return bytes(i & 0xFF for i in range(n))


# ---------------------------------------------------------------- canon
def test_canon_prints_strided_form_and_plan(tf):  # test_cli.cpp:70-83
    f = tf("cuboid.types", CUBOID)
    code, out, _ = run("canon", f)
    assert code == 0
    assert out == ("sb start=0 counts=[400,13,47] strides=[1,256,131072]\n"
                   "plan w=16 block=(32,16,2) grid=(1,1,24) strategy=iterate\n")
    assert run("canon", f)[1] == out  # byte-stable


def test_canon_named_byte(tf):  # test_cli.cpp:85-93
    code, out, _ = run("canon", tf("b.types", "type t = named(byte)\ncommit t\n"))
    assert code == 0
    assert out == "sb start=0 counts=[1] strides=[1]\nplan w=1 block=(1,1,1) grid=(1,1,1) strategy=gridz\n"


def test_canon_empty(tf):  # test_cli.cpp:95-102
    code, out, _ = run("canon", tf("e.types", "type t = vector(0, 4, 8, float)\ncommit t\n"))
    assert (code, out) == (0, "sb empty\n")


def test_canon_unsupported_exit_2(tf):  # test_cli.cpp:104-111
    code, out, _ = run("canon", tf("u.types", "type t = vector(2, 1, 0, byte)\ncommit t\n"))
    assert (code, out) == (2, "unsupported blocks=1\n")


def test_undefined_names_diagnosed(tf):  # test_cli.cpp:113-120
    code, _, err = run("canon", tf("bad.types", "type t = contiguous(4, nosuch)\ncommit t\n"))
    assert code == 1 and "nosuch" in err and "line 1" in err


def test_second_commit_or_missing_commit(tf):  # test_cli.cpp:318-326
    assert run("canon", tf("two.types", "type a = named(byte)\ncommit a\ncommit a\n"))[0] == 1
    assert run("canon", tf("none.types", "type a = named(byte)\n"))[0] == 1


# ---------------------------------------------------------------- flatten
def test_flatten_pairs(tf):  # test_cli.cpp:122-129
    assert run("flatten", tf("v.types", VEC)) == (0, "0 16\n32 16\n64 16\n", "")


def test_flatten_empty(tf):  # test_cli.cpp:131-137
    code, out, _ = run("flatten", tf("e.types", "type t = contiguous(0, byte)\ncommit t\n"))
    assert code == 0 and out == ""


def test_flatten_marks_overlap(tf):  # test_cli.cpp:139-148
    assert run("flatten", tf("o.types", OVERLAP))[:2] == (0, "0 3472\n# overlap\n")


# ---------------------------------------------------------------- beyond the reference
def test_typefile_indexed_struct_resized(tf, sp):
    """the engine's extra constructors in the type-file language: a regular
    indexed type canonicalises, an irregular one reports the block-list form
    (exit 2, like the reference's unsupported forms), struct + resized
    flatten to the MPI typemap (oracle/typemap.py)"""
    from oracle import typemap as tm
    reg = "type d = named(double)\ntype t = indexed([2,2,2], [0,5,10], d)\ncommit t\n"
    code, out, _ = run("canon", tf("reg.types", reg))
    assert code == 0 and out.startswith("sb start=0 counts=[16,3] strides=[1,40]\n")
    irr = "type t = hindexed([16,24,8], [8,40,80], byte)\ncommit t\n"
    assert run("canon", tf("irr.types", irr))[:2] == (2, "unsupported blocks=3\n")
    src = ("type d = named(double)\ntype s = struct([1,2], [0,8], [int, d])\n"
           "type r = resized(s, 0, 32)\ntype v = contiguous(4, r)\ncommit v\n")
    code, out, _ = run("flatten", tf("s.types", src))
    _, _, _, runs = tm.typemap(("contiguous", 4, ("resized", 0, 32,
                                                  ("struct", [1, 2], [0, 8], [("named", 4), ("named", 8)]))))
    norm, _ = tm.normalized(runs)
    assert code == 0 and out == "".join(f"{o} {n}\n" for o, n in norm)
    code, _, err = run("canon", tf("bad.types", "type t = struct([1], [0, 8], [byte])\ncommit t\n"))
    assert code == 1 and "line 1" in err


# ---------------------------------------------------------------- choose
def test_choose_prints_method_and_times():  # test_cli.cpp:226-245
    code, out, _ = run("choose", "--object-bytes", 4194304, "--block-bytes", 16, "--profile", PROFILE)
    assert code == 0 and out.startswith("method=device ")
    for k in ("t_oneshot=", "t_device=", "t_staged="):
        assert k in out
    assert run("choose", "--object-bytes", 4194304, "--block-bytes", 16, "--profile", PROFILE)[1] == out
    small = run("choose", "--object-bytes", 256, "--block-bytes", 16, "--profile", PROFILE)[1]
    assert small.startswith("method=oneshot ")


def test_choose_matches_reference_model_bitwise():
    """the printed times are the reference's (model_golden.json) to %.6e"""
    queries = json.load(open(os.path.join(GOLD, "model_golden.json")))["base"]  # default.profile
    names = {0: "oneshot", 1: "device", 2: "staged"}
    for q in [q for q in queries if q["status"] == 0][::61][:12]:
        o, b = q["o"], q["b"]
        code, out, _ = run("choose", "--object-bytes", o, "--block-bytes", b, "--profile", PROFILE)
        assert code == 0
        want = (f"method={names[q['method']]} t_oneshot={q['t_oneshot']:.6e} t_device={q['t_device']:.6e} "
                f"t_staged={q['t_staged']:.6e}\n")
        assert out == want


def test_choose_zero_pack_profile(tf):  # test_cli.cpp:247-266
    text = ("curve cpu_cpu\n64 1.3e-6\n4194304 4e-4\ncurve gpu_gpu\n64 6e-6\n4194304 5e-4\n"
            "curve d2h\n64 7e-6\n4194304 2e-4\ncurve h2d\n64 7e-6\n4194304 2e-4\n")
    for s in ("gpu_pack", "gpu_unpack", "host_pack", "host_unpack"):
        text += f"surface {s}\n64 8 0\n64 4096 0\n4194304 8 0\n4194304 4096 0\n"
    code, out, _ = run("choose", "--object-bytes", 128, "--block-bytes", 8, "--profile", tf("zero.profile", text))
    assert code == 0 and out.startswith("method=oneshot ")


def test_choose_without_profile():  # test_cli.cpp:268-273
    code, _, err = run("choose", "--object-bytes", 64, "--block-bytes", 8, "--profile", "/nonexistent/profile")
    assert code == 1 and err


def test_usage_errors():
    assert run()[0] == 1
    assert run("frobnicate")[0] == 1
    assert run("pack", "a")[0] == 1
    assert run("choose", "--object-bytes", 1)[0] == 1
    assert run("--help")[0] == 0


# ---------------------------------------------------------------- type files
def _typefile(prog):
    """a reference-corpus type program (oracle/ref_harness.cpp layout) as a
    type file, one statement per node, innermost first"""
    lines, it, ids = [], iter(prog), iter(range(1 << 30))
    kinds = ["byte", "int", "float", "double"]

    def rec():
        tag = next(it)
        if tag == 0:
            return kinds[next(it)]
        name = f"t{next(ids)}"
        if tag == 1:
            c = next(it)
            inner = rec()
            lines.append(f"type {name} = contiguous({c}, {inner})")
        elif tag in (2, 3):
            c, bl, s = next(it), next(it), next(it)
            inner = rec()
            lines.append(f"type {name} = {'vector' if tag == 2 else 'hvector'}({c}, {bl}, {s}, {inner})")
        else:
            nd, _order = next(it), next(it)
            sz = [next(it) for _ in range(nd)]
            sub = [next(it) for _ in range(nd)]
            off = [next(it) for _ in range(nd)]
            inner = rec()
            lst = lambda v: "[" + ", ".join(map(str, v)) + "]"
            lines.append(f"type {name} = subarray({nd}, {lst(sz)}, {lst(sub)}, {lst(off)}, {inner})")
        return name

    top = rec()
    if top in kinds:
        lines.append(f"type top = named({top})")
        top = "top"
    return "# generated from a reference corpus program\n" + "\n".join(lines) + f"\ncommit {top}\n"


def test_typefile_corpus_matches_reference(sp, corpus):
    """every reference-corpus definition, written as a type file, commits to
    the reference's canonical StridedBlock / size / extent / overlap"""
    n = 0
    for e in corpus:
        want = e["ref"]
        if want.get("status", 0) != 0:
            continue
        r = sp.parse_type_file(_typefile(e["prog"]))
        ct = sp.commit_type(r.def_)
        assert (ct.size, ct.extent, ct.span, int(ct.overlapping)) == (want["size"], want["extent"], want["span"],
                                                                     want["overlapping"])
        if want["form"] == 0:
            assert ct.canon == sp.StridedBlock(want["start"], tuple(want["counts"]), tuple(want["strides"]))
        n += 1
    assert n > 500


def test_typefile_diagnostics(sp):
    cases = {
        "type a = named(byte)\ncommit a\ncommit a\n": "line 3: statement after commit",
        "type a = named(byte)\n": "type file has no commit statement",
        "type 1a = named(byte)\ncommit 1a\n": "line 1: invalid type name '1a'",
        "type byte = named(int)\ncommit byte\n": "line 1: type name 'byte' is already in use",
        "type a = named(byte)\ntype a = named(int)\ncommit a\n": "line 2: type name 'a' is already in use",
        "type a = vector(1, 2, byte)\ncommit a\n": "line 1: vector takes 4 arguments",
        "type a = contiguous(x, byte)\ncommit a\n": "line 1: expected an integer, got 'x'",
        "type a = subarray(1, 4, [1], [0], byte)\ncommit a\n": "line 1: expected a [..] list, got '4'",
        "type a = subarray(1, [4, [1], [0], byte)\ncommit a\n": "line 1: unbalanced '['",
        "type a = named(quad)\ncommit a\n": "line 1: unknown kind 'quad'",
        "type a = stack(4, byte)\ncommit a\n": "line 1: unknown constructor 'stack'",
        "type a = contiguous(-1, byte)\ncommit a\n": "line 1: contiguous: count must be >= 0",
        "typedef a = named(byte)\n": "line 1: expected 'type' or 'commit', got 'typedef'",
        "type a named(byte)\n": "line 1: expected 'type <name> = <constructor>'",
        "commit\n": "line 1: commit takes exactly one name",
        "type a = named(byte)\ncommit b\n": "line 2: undefined type 'b'",
    }
    for text, msg in cases.items():
        with pytest.raises(sp.ParseError) as ei:
            sp.parse_type_file(text)
        assert str(ei.value).endswith(msg) or msg in str(ei.value), (text, str(ei.value))
    # comments, blank lines and a named alias of a kind
    r = sp.parse_type_file("\n  # header\ntype d = named(double)   # eight bytes\n\ncommit d\n")
    assert r.name == "d" and r.def_.size() == 8


# ---------------------------------------------------------------- GPU commands
@pytest.mark.gpu
def test_pack_and_unpack_move_file_bytes(tf, cuda):  # test_cli.cpp:150-185
    types = tf("v.types", VEC)
    inp = tf("in.bin", ramp(96))
    out = str(tf.dir / "packed.bin")
    assert run("pack", types, inp, out)[0] == 0
    packed = open(out, "rb").read()
    want = b"".join(bytes(range(b, b + 16)) for b in (0, 32, 64))
    assert packed == want
    rest = str(tf.dir / "restored.bin")
    assert run("unpack", types, out, rest)[0] == 0
    restored = open(rest, "rb").read()
    assert len(restored) == 80
    orig = ramp(96)
    for b in (0, 32, 64):
        assert restored[b:b + 16] == orig[b:b + 16]
    assert restored[20] == 0  # gaps zero-filled


@pytest.mark.gpu
def test_pack_count_places_objects_one_extent_apart(tf, cuda):  # test_cli.cpp:187-212
    types = tf("v.types", VEC)
    inp = tf("in.bin", ramp(160))
    out = str(tf.dir / "packed.bin")
    assert run("pack", types, inp, out, "--count", 2)[0] == 0
    packed = open(out, "rb").read()
    assert len(packed) == 96
    for j in range(2):
        for i in range(3):
            assert packed[j * 48 + i * 16:j * 48 + i * 16 + 16] == bytes(range(j * 80 + i * 32, j * 80 + i * 32 + 16))
    rest = str(tf.dir / "restored.bin")
    assert run("unpack", types, out, rest, "--count", 2)[0] == 0
    assert len(open(rest, "rb").read()) == 160


@pytest.mark.gpu
def test_pack_reports_undersized_input(tf, cuda):  # test_cli.cpp:214-222
    code, _, err = run("pack", tf("v.types", VEC), tf("in.bin", ramp(10)), str(tf.dir / "o.bin"))
    assert code == 1 and "need" in err


@pytest.mark.gpu
def test_unpack_refuses_overlap(tf, cuda):  # test_cli.cpp:224-234
    code, _, err = run("unpack", tf("o.types", OVERLAP), tf("in.bin", b"\x01" * 5200), str(tf.dir / "o.bin"))
    assert code == 1 and "overlap" in err


@pytest.mark.gpu
def test_pack_file_bytes_match_oracle(tf, cuda, orc):
    """a 3-D subarray of random bytes through the CLI equals the oracle's pack"""
    prog = [4, 3, 0, 96, 40, 24, 24, 16, 8, 8, 4, 2, 0, 2]
    types = tf("s.types", _typefile(prog))
    rng = np.random.default_rng(3)
    c = orc.commit(prog)
    src = rng.integers(0, 256, 2 * c.extent, dtype=np.uint8)
    inp = tf("in.bin", src.tobytes())
    out = str(tf.dir / "p.bin")
    assert run("pack", types, inp, out, "--count", 2)[0] == 0
    want = np.zeros(2 * c.size, np.uint8)
    st, _ = orc.pack(prog, src, 2, want, 0)
    assert st == 0 and open(out, "rb").read() == want.tobytes()


@pytest.mark.gpu
def test_halo_matches_reference_reports(cuda):  # test_cli.cpp:289-312 + golden reports
    gold = json.load(open(os.path.join(GOLD, "halo_golden.json")))["reports"]
    for rep in gold[:6]:
        args = ["halo", "--ranks", ",".join(map(str, rep["ranks"])), "--interior",
                ",".join(map(str, rep["interior"])), "--radius", rep["radius"], "--element-bytes", rep["elem"],
                "--profile", PROFILE]
        code, out, err = run(*args)
        assert code == 0, err
        tot = rep["pack"] + rep["alltoallv"] + rep["unpack"]
        want = (f"pack,{rep['pack']:.6e}\nalltoallv,{rep['alltoallv']:.6e}\nunpack,{rep['unpack']:.6e}\n"
                f"summary,total={tot:.6e},bytes={rep['bytes']},verify=PASS\n")
        assert out == want
        assert "verified" in err
        assert run(*args)[1] == out  # byte-stable


def test_halo_rejects_oversized_radius():  # test_cli.cpp:314-316
    code, _, err = run("halo", "--ranks", "1,1,1", "--interior", "4,4,4", "--radius", 3, "--profile", PROFILE)
    assert code == 1 and err


@pytest.mark.gpu
def test_profile_gen_emits_loadable_profile(tf, cuda, sp):  # test_cli.cpp:275-287
    import paper_2012_14363_b200.model as M
    out = str(tf.dir / "m.profile")
    assert run("profile-gen", "--out", out)[0] == 0
    p = M.load_profile_file(out)
    assert run("profile-gen", "--out", out)[0] == 0  # overwrite
    M.load_profile_file(out)
    assert p is not None


def test_flatten_matches_oracle_on_corpus(sp, orc, corpus):
    """sp_type_flatten (the CLI's `flatten`) == the oracle's normalized block
    list (block_list.hpp:44-61 over :67-121) on reference-corpus definitions
    small enough to enumerate"""
    n = 0
    for e in corpus:
        r = e["ref"]
        if r["status"] != 0 or r["size"] > (1 << 16):
            continue
        st, blocks, overlap = orc.flatten(e["prog"])
        assert st == 0
        got = sp.flatten(sp.from_program(e["prog"]))
        assert [(b.offset, b.length) for b in got.blocks] == blocks, e["prog"]
        assert got.overlap == overlap
        n += 1
    assert n > 300


def test_flatten_matches_live_reference(sp, ref):
    """against the reference compiled in place, on a fresh corpus"""
    progs = ref.corpus(0xF1A7, 200, 0)
    n = 0
    for prog in progs:
        st, blocks, overlap = ref.flatten(prog)
        if st != 0 or sum(l for _, l in blocks) > (1 << 16):
            continue
        got = sp.flatten(sp.from_program(prog))
        assert [(b.offset, b.length) for b in got.blocks] == blocks, prog
        assert got.overlap == overlap
        n += 1
    assert n > 50


def test_enumerate_and_normalize_match_flatten(sp, corpus):
    """block_list.hpp: enumerate_blocks(canonical form) == flatten(definition)
    for strided definitions (translate + canonicalisation preserve the byte
    set), and normalize_blocks of the definition's runs is idempotent"""
    n = 0
    for e in corpus:
        r = e["ref"]
        if r["status"] != 0 or r["form"] != 0 or r["size"] > (1 << 14) or r["overlapping"]:
            continue
        d = sp.from_program(e["prog"])
        ct = sp.commit_type(d)
        got = sp.flatten_oracle(d)
        assert sp.enumerate_blocks(ct.canon) == got, e["prog"]
        assert sp.normalize_blocks(got.blocks) == got
        n += 1
    assert n > 100
    assert sp.normalize_blocks([(8, 4), (0, 4), (2, 4), (12, 0)]) == sp.BlockList(
        (sp.Block(0, 6), sp.Block(8, 4)), True)
