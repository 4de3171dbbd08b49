# ncu evidence: bench launch list + full captures of the halo batch kernels (copied to profiles/ by hand)
set -o pipefail
mkdir -p gpurun_out
timeout 900 python bench.py 2>gpurun_out/bench.err | tee gpurun_out/bench.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_batchp -s 1 -c 1 -o gpurun_out/r01_full_halo_direct python scripts/halo_one.py direct 3 > gpurun_out/halo_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_batchp -s 2 -c 2 -o gpurun_out/r01_full_halo_fused python scripts/halo_one.py fused 3 >> gpurun_out/halo_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 0 > gpurun_out/bench_ncu.log 2>&1
timeout 300 python scripts/halo_regions.py 7 2>&1 | tee gpurun_out/halo_regions.json
tail -2 gpurun_out/halo_ncu.log
