"""Regenerates the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in a container that has /root/reference (it drives
oracle/_ref/libstridepack_ref.so, the unmodified reference headers compiled in
place by oracle/Makefile):

    python tests/golden/make_golden.py

Outputs (committed, small, consumed by tests on the GPU box where the
reference tree does not exist):
  corpus.json        reference-generated definitions (tests/test_util.hpp
                     random_def driven like acceptance.cpp:59-69 / :175-178)
                     with the reference's commit_type() results
  pack_digests.json  sha256 of reference pack/unpack outputs on seeded inputs
  default.profile    proj/data/default.profile after the reference's own
                     load_profile -> save_profile round trip
  model_golden.json  reference choose_method + model times on a query grid
  halo_golden.json   reference halo region programs and run_exchange reports
"""
from __future__ import annotations

import ctypes as C  # noqa: F401
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import reference  # noqa: E402

REF_PROFILE = "/root/reference/proj/data/default.profile"


def commit_record(R, prog):
    c = R.commit(prog)
    rec = {"status": c.status}
    if c.status == 0:
        rec.update(form=c.form, size=c.size, extent=c.extent, span=c.span,
                   overlapping=int(c.overlapping), n_fallback_runs=c.n_fallback_runs)
        if c.form == 0:
            rec.update(start=c.start, counts=c.counts, strides=c.strides, word=c.word,
                       block=list(c.block), grid=list(c.grid), strategy=c.strategy,
                       rounds=c.simplify_rounds)
    return rec


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make_corpus(R):
    out = []
    for name, seed, count, mode in [("acceptance", 0xACCE, 1000, 0),
                                    ("roundtrip", 0x4CAFE, 500, 1),
                                    ("default", 5, 500, 2)]:
        for i, prog in enumerate(R.corpus(seed, count, mode)):
            out.append({"set": name, "i": i, "prog": prog, "ref": commit_record(R, prog)})
    return out


def make_pack_digests(R, corpus):
    rows = []
    k = 0
    for e in corpus:
        ref = e["ref"]
        if ref["status"] != 0 or ref["size"] == 0 or ref["size"] > (1 << 16):
            continue
        k += 1
        if k % 3:
            continue
        prog = e["prog"]
        seed = 1000 + len(rows)
        incount = 1 + seed % 3
        position = seed % 5
        rng = np.random.default_rng(seed)
        src_len = (incount - 1) * ref["extent"] + ref["span"]
        src = rng.integers(0, 256, src_len, dtype=np.uint8)
        dst = np.zeros(position + incount * ref["size"], np.uint8)
        st, npos = R.pack(prog, src, incount, dst, position)
        row = {"prog": prog, "seed": seed, "incount": incount, "position": position,
               "pack_status": st, "packed": sha(dst[position:])}
        if st == 0 and not ref["overlapping"]:
            back = np.full(src_len, 0xCD, np.uint8)
            st2, _ = R.unpack(prog, dst, position, incount, back)
            row["unpack_status"] = st2
            row["unpacked"] = sha(back)
        rows.append(row)
    return rows


def main():
    R = reference()
    if R is None:
        raise SystemExit("oracle/_ref is not built: run `make -C oracle` where /root/reference exists")
    corpus = make_corpus(R)
    with open(os.path.join(HERE, "corpus.json"), "w") as f:
        json.dump(corpus, f, separators=(",", ":"))
    digests = make_pack_digests(R, corpus)
    with open(os.path.join(HERE, "pack_digests.json"), "w") as f:
        json.dump(digests, f, separators=(",", ":"))
    print(f"corpus: {len(corpus)} defs, pack digests: {len(digests)}")
    try:
        sys.path.insert(0, HERE)
        import make_golden_model
        make_golden_model.main(R)
    except ImportError:
        pass


if __name__ == "__main__":
    main()
