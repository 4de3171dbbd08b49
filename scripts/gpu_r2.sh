set -o pipefail
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.log
for m in direct fused copy; do python scripts/halo_one.py $m 20; done 2>&1 | tee gpurun_out/halo_one.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_batch -s 2 -c 3 -o gpurun_out/halo_direct python scripts/halo_one.py direct 2 > gpurun_out/halo_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_batch -s 4 -c 2 -o gpurun_out/halo_fused2 python scripts/halo_one.py fused 3 >> gpurun_out/halo_ncu.log 2>&1
tail -3 gpurun_out/halo_ncu.log
timeout 900 python bench.py 2>gpurun_out/bench.err | tee gpurun_out/bench.json
