set -o pipefail
mkdir -p gpurun_out
timeout 300 python scripts/halo_regions.py 5 2>&1 | tee gpurun_out/halo_regions.txt
for m in direct fused; do python scripts/halo_one.py $m 20; done 2>&1 | tee gpurun_out/halo_one.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_batch -s 1 -c 1 -o gpurun_out/halo_direct2 python scripts/halo_one.py direct 3 > gpurun_out/halo_ncu.log 2>&1
timeout 1200 python -m pytest tests/test_halo.py tests/test_rt.py tests/test_pack_gpu.py -m gpu -q -x 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.log
