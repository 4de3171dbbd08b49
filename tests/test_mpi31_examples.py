"""Known answers from the MPI-3.1 standard for the datatypes the reference
does not have: the worked typemap examples of
section 4.1.2 under MPI_TYPE_CONTIGUOUS, MPI_TYPE_VECTOR, MPI_TYPE_INDEXED
and MPI_TYPE_CREATE_STRUCT, transcribed in tests/golden/
mpi31_typemap_examples.json. They pin both the typemap restatement the
random-description tests trust (oracle/typemap.py) and the engine itself to
an external source.

CPU: the restatement and the engine's size / lb / extent / flattened runs
against the standard's typemaps. GPU: pack of two objects in typemap order
(MPI_Pack's order: the indexed example packs its block at displacement 64
first) and unpack into a sentinel buffer, against a gather / scatter
written directly from the standard's typemap.
"""
import json
import os

import numpy as np
import pytest

from oracle import typemap as tm

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "mpi31_typemap_examples.json")
with open(GOLDEN) as f:
    G = json.load(f)
EXAMPLES = G["examples"]
NBYTES = G["bytes"]


def _desc(x):
    """JSON description -> the nested tuples of oracle/typemap.py"""
    if not (isinstance(x, list) and x and isinstance(x[0], str)):
        return x
    out = [x[0]]
    for v in x[1:]:
        if isinstance(v, list) and v and isinstance(v[0], list):
            out.append([_desc(m) for m in v])
        elif isinstance(v, list) and v and isinstance(v[0], str):
            out.append(_desc(v))
        else:
            out.append(v)
    return tuple(out)


def _std_runs(ex):
    """the standard's typemap as byte runs in typemap order, adjacent merged"""
    runs = []
    for kind, disp in ex["typemap"]:
        n = NBYTES[kind]
        if runs and runs[-1][0] + runs[-1][1] == disp:
            runs[-1] = (runs[-1][0], runs[-1][1] + n)
        else:
            runs.append((disp, n))
    return runs


def _gather(src, runs, count, extent):
    return np.concatenate([src[j * extent + o: j * extent + o + n] for j in range(count) for o, n in runs])


@pytest.mark.parametrize("ex", EXAMPLES, ids=[e["constructor"] for e in EXAMPLES])
def test_restatement_matches_standard(ex):
    size, lb, ext, runs = tm.typemap(_desc(ex["desc"]))
    assert (size, lb, ext) == (ex["size"], ex["lb"], ex["extent"])
    assert runs == _std_runs(ex)


@pytest.mark.parametrize("ex", EXAMPLES, ids=[e["constructor"] for e in EXAMPLES])
def test_engine_matches_standard(sp, ex):
    t = tm.build(sp, _desc(ex["desc"]))
    assert (t.size(), t.lb(), t.extent()) == (ex["size"], ex["lb"], ex["extent"])
    norm, overlap = tm.normalized(_std_runs(ex))
    fl = sp.flatten(t)
    assert [(b.offset, b.length) for b in fl.blocks] == norm and fl.overlap == overlap
    c = sp.commit_type(t)
    assert (c.size, c.extent) == (ex["size"], ex["extent"])


@pytest.mark.gpu
@pytest.mark.parametrize("ex", EXAMPLES, ids=[e["constructor"] for e in EXAMPLES])
def test_pack_unpack_in_standard_order(sp, cuda, ex):
    torch = cuda
    c = sp.commit_type(tm.build(sp, _desc(ex["desc"])))
    runs, count, ext = _std_runs(ex), 2, ex["extent"]
    rng = np.random.default_rng(31)
    host = rng.integers(0, 256, count * ext + 64, dtype=np.uint8)
    want = _gather(host, runs, count, ext)
    assert want.size == count * ex["size"]
    dst = torch.zeros(want.size, dtype=torch.uint8, device="cuda")
    pos = sp.pack(torch.from_numpy(host).cuda(), c, count, dst, 0, sync=True)
    assert pos == want.size
    assert np.array_equal(dst.cpu().numpy(), want), ex["name"]
    back = torch.full((host.size,), 0xA5, dtype=torch.uint8, device="cuda")
    sp.unpack(dst, 0, c, count, back, sync=True)
    exp = np.full(host.size, 0xA5, np.uint8)
    for j in range(count):
        for o, n in runs:
            exp[j * ext + o: j * ext + o + n] = host[j * ext + o: j * ext + o + n]
    assert np.array_equal(back.cpu().numpy(), exp), ex["name"]
