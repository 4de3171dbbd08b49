timeout 120 python scripts/halo_exp.py
timeout 600 python -m pytest tests/test_rt.py tests/test_halo.py -m gpu -q 2>&1 | tail -2
