timeout 900 python -m pytest tests/test_rt.py tests/test_halo.py -m gpu -x -q 2>&1 | tail -30 | tee gpurun_out/pytest_rt.log
