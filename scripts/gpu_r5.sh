set -o pipefail
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_rt.py tests/test_mpi.py -m gpu -q -x 2>&1 | tail -30 | tee gpurun_out/pytest_rt.log
