timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ -c 1 -o gpurun_out/r01_full_unpack_e0_1 python scripts/prof_cfg2.py --e0 1 --k 64 --reps 1 --mode unpack > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ -c 1 -o gpurun_out/r01_full_pack_e0_512 python scripts/prof_cfg2.py --e0 512 --k 64 --reps 1 --mode pack > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ -c 1 -o gpurun_out/r01_full_pack_e0_32 python scripts/prof_cfg2.py --e0 32 --k 64 --reps 1 --mode pack > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
