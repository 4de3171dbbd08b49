timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.log
timeout 600 python scripts/halo_bench.py 2>&1 | tee gpurun_out/halo_bench.txt
