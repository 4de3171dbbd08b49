#!/bin/bash
# round 2: graph capture with ranks sharing a GPU (one-warp device-numbered
# wait kernel), the halo/runtime/MPI suites in both flag-wait modes
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export TEMPI_TIMEOUT=60
timeout 1500 python -m pytest -q -m gpu tests/test_halo.py tests/test_rt.py tests/test_mpi.py > gpurun_out/r02ag_stream.log 2>&1
echo "rc=$?" >> gpurun_out/r02ag_stream.log
TEMPI_FLAG_WAIT=kernel timeout 1500 python -m pytest -q -m gpu tests/test_halo.py tests/test_rt.py -k "graph or halo" > gpurun_out/r02ag_kernel.log 2>&1
echo "rc=$?" >> gpurun_out/r02ag_kernel.log
tail -n 3 gpurun_out/r02ag_stream.log gpurun_out/r02ag_kernel.log; grep -E "^FAILED" gpurun_out/r02ag_*.log | head
