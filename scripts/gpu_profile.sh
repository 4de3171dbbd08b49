# ncu evidence for the shipped kernels: bench launch list + full captures of
# the halo batch kernels and a single typed copy (copy to profiles/ by hand)
set -o pipefail
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_batchp -s 1 -c 1 -o gpurun_out/r01_full_halo_direct_copy python scripts/halo_one.py direct 3 > gpurun_out/ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_batchp -s 2 -c 2 -o gpurun_out/r01_full_halo_fused_pack_unpack python scripts/halo_one.py fused 3 >> gpurun_out/ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_job -c 1 -o gpurun_out/r01_full_copy_e0_512 python -c "
import sys, math; sys.path.insert(0, '.')
import torch, paper_2012_14363_b200 as sp
e0, n = 512, 64 << 20
rows = n // e0; e2 = 2 ** (int(math.log2(rows)) // 2); e1 = rows // e2
ct = sp.commit_type(sp.from_program([4, 3, 0, max(2 * e0, 64), 2 * e1, e2, e0, e1, e2, 0, 0, 0, 0, 0]))
a = torch.empty(ct.span, dtype=torch.uint8, device='cuda'); b = torch.empty_like(a)
sp.copy(a, ct, 1, b, ct, 1, sync=True)
" >> gpurun_out/ncu.log 2>&1
tail -3 gpurun_out/ncu.log
ls -la gpurun_out/*.ncu-rep
