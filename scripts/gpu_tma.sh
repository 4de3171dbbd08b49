timeout 900 python -m pytest tests/test_pack_gpu.py -m gpu -x -q -k "tma" 2>&1 | tail -15
for kern in 1 4; do timeout 300 python scripts/prof_cfg2.py --e0 512,256,128,64,32,16 --k 64 --reps 5 --kernel $kern; done 2>&1 | tee gpurun_out/tma_vs_words.txt
timeout 600 ncu --set full --clock-control none -k regex:k_tma -c 4 -o gpurun_out/prof_tma python scripts/prof_cfg2.py --e0 512,32 --k 64 --reps 1 --kernel 4 > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
