timeout 900 ./tools/measure_profile gpurun_out/b200.profile 25 2>&1 | tail -6
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_batch -c 4 -o gpurun_out/prof_batch python scripts/halo_bench.py > gpurun_out/prof_batch.log 2>&1; tail -2 gpurun_out/prof_batch.log
