"""Single-process halo exchange timings (all ranks on one GPU)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2012_14363_b200.halo as H
import paper_2012_14363_b200.model as M
prof = M.load_profile_file(os.path.join(ROOT, "tests", "golden", "default.profile"))
for ranks in [(1, 1, 1), (2, 1, 1), (2, 2, 1), (2, 2, 2)]:
    for method in (H.FUSED, H.COPY):
        cfg = H.HaloConfig(ranks, (256, 256, 256), 2, 32)
        r = H.run_exchange(cfg, prof, method=method, iters=10)
        n = ranks[0] * ranks[1] * ranks[2]
        hbm = 4 * 25561088 * n
        tot = r.measured_pack_seconds + r.measured_exchange_seconds + r.measured_unpack_seconds
        print(json.dumps({"ranks": ranks, "method": ["fused", "copy"][method], "verified": r.verified,
                          "pack_us": round(r.measured_pack_seconds * 1e6, 1),
                          "xchg_us": round(r.measured_exchange_seconds * 1e6, 1),
                          "unpack_us": round(r.measured_unpack_seconds * 1e6, 1),
                          "total_us": round(tot * 1e6, 1),
                          "hbm_GBps": round(hbm / tot / 1e9, 1)}), flush=True)
