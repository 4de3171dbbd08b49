"""One-rank halo exchange (BASELINE config 5 geometry) for profiling."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2012_14363_b200.halo as H
import paper_2012_14363_b200.model as M
method = {"fused": H.FUSED, "copy": H.COPY, "direct": H.DIRECT}.get(sys.argv[1] if len(sys.argv) > 1 else "fused")
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
prof = M.load_profile_file(os.path.join(ROOT, "tests", "golden", "default.profile"))
r = H.run_exchange(H.HaloConfig((1, 1, 1), (256, 256, 256), 2, 32), prof, method=method, iters=iters)
print(json.dumps({"verified": r.verified, "pack_us": r.measured_pack_seconds * 1e6,
                  "xchg_us": r.measured_exchange_seconds * 1e6, "unpack_us": r.measured_unpack_seconds * 1e6}))
