timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -8 | tee gpurun_out/pytest_all.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for kern in 1 4; do timeout 300 python scripts/prof_cfg2.py --e0 512,256,128,64,32 --k 64 --reps 5 --kernel $kern; done 2>&1 | tee gpurun_out/tma_vs_words_clean.txt
