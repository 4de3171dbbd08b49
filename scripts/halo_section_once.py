import sys, json, os, uuid
sys.path.insert(0, os.getcwd())
import torch
from tools.bench_parts import halo_section
torch.cuda.set_device(0)
for _ in range(2):
    h = halo_section(torch, 0, 1, 0, "hs" + uuid.uuid4().hex[:8])
    print(json.dumps({"direct": h["direct_us"]["iteration"], "fused": h["fused_us"], "mpi_w": h["mpi_alltoallw_us"], "ok": h["verified"]}))
