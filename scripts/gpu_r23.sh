set -o pipefail
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_mpi.py tests/test_rt.py -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/pytest_mpi_rt.log
bash scripts/gpu_sanitize2.sh
