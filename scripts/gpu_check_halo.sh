# halo plans + neighbour collectives: distributed tests + the bench's one-rank halo section
set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_rt.py tests/test_halo.py tests/test_mpi.py -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/pytest_halo.log
timeout 300 python tools/bench_parts.py 2>&1 | tail -1 | tee gpurun_out/halo_section.json
