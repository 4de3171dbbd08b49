for k in 8 32 64; do timeout 300 python scripts/prof_cfg2.py --e0 512,128,32,16,8,1 --k $k --reps 5 --copy; done 2>&1 | tee gpurun_out/prof1_times.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ -c 12 -o gpurun_out/prof1 python scripts/prof_cfg2.py --e0 512,32,8,1 --k 32 --reps 1 > gpurun_out/prof1_ncu.log 2>&1
tail -5 gpurun_out/prof1_ncu.log
