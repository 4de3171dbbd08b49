# round-end evidence: tests, smoke, bench (+ reference arm), launch list,
# TMA E0=64 capture, and full captures of the run-table kernels
bash scripts/gpu_final.sh > gpurun_out/final.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_runs -c 1 -o gpurun_out/r01_full_runs_pack_1k python scripts/prof_runs.py --block 1024 > gpurun_out/prof_runs.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_runs_multi -c 1 -o gpurun_out/r01_full_runs_multi python scripts/unstructured_halo.py > gpurun_out/prof_runs_multi.log 2>&1
tail -5 gpurun_out/final.log
