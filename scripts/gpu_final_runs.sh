bash scripts/gpu_final.sh > gpurun_out/final.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_runs -c 1 -o gpurun_out/r01_full_runs_pack_1k python scripts/prof_runs.py --block 1024 > gpurun_out/prof_runs.log 2>&1
tail -5 gpurun_out/final.log
