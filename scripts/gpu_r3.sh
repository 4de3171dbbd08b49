set -o pipefail
mkdir -p gpurun_out
for m in direct fused; do python scripts/halo_one.py $m 20; done 2>&1 | tee gpurun_out/halo_one.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_batch -s 1 -c 2 -o gpurun_out/halo_direct python scripts/halo_one.py direct 3 > gpurun_out/halo_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_batch -s 4 -c 2 -o gpurun_out/halo_fused3 python scripts/halo_one.py fused 3 >> gpurun_out/halo_ncu.log 2>&1
tail -3 gpurun_out/halo_ncu.log
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.log
