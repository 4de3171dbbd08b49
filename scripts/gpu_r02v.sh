#!/bin/bash
# round 2: stale IPC mappings evicted on cudaErrorAlreadyMapped (a peer that
# freed and re-made a receive buffer at the same address) -- the all-to-all
# reproducer, then the full GPU suite
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python -m pytest -q -m gpu tests/test_mpi.py tests/test_interpose.py -k "alltoall" > gpurun_out/r02v_alltoall.log 2>&1
echo "rc=$?" >> gpurun_out/r02v_alltoall.log
tail -n 3 gpurun_out/r02v_alltoall.log
timeout 2400 python -m pytest -q -m gpu tests > gpurun_out/r02v_pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r02v_pytest_gpu.log
tail -n 4 gpurun_out/r02v_pytest_gpu.log
