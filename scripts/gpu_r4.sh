set -o pipefail
mkdir -p gpurun_out
timeout 300 python scripts/halo_regions.py 5 2>&1 | tee gpurun_out/halo_regions.txt
timeout 900 python -m pytest tests/test_rt.py tests/test_halo.py tests/test_cli.py -m gpu -q -x 2>&1 | tail -30 | tee gpurun_out/pytest_rt.log
