#!/bin/bash
# round 2: set completions (Waitany/Waitsome/Testall/Testany/Request_free) in
# the engine's MPI, the stand-in MPI and the interposer
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -m gpu tests/test_mpi.py tests/test_interpose.py > gpurun_out/r02y_mpi.log 2>&1
echo "rc=$?" >> gpurun_out/r02y_mpi.log
tail -n 4 gpurun_out/r02y_mpi.log; grep -E "^FAILED|FAIL rank" gpurun_out/r02y_mpi.log | head
