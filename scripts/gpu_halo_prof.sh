mkdir -p gpurun_out
python scripts/halo_one.py fused 20 | tee gpurun_out/halo_one.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_batch -s 4 -c 2 -o gpurun_out/halo_batch python scripts/halo_one.py fused 3 > gpurun_out/halo_ncu.log 2>&1
tail -3 gpurun_out/halo_ncu.log
