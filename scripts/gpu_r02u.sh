#!/bin/bash
# round 2: why the engine's alltoallv (dense send -> strided receive) fails
# at 2+ ranks (verbose), then the kernel-choice counter pass again
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
PKG=paper_2012_14363_b200
gcc -O2 -Iinclude -I/usr/local/cuda/include tests/native/mpi_alltoall.c -o /tmp/a2a -L$PKG -ltempi_b200 -lstridepack_b200 \
  -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/$PKG
TEMPI_VERBOSE=1 timeout 120 python tools/tempirun.py -n 2 --timeout 100 /tmp/a2a > gpurun_out/r02u_a2a_verbose.log 2>&1
echo "rc=$?" >> gpurun_out/r02u_a2a_verbose.log
cat gpurun_out/r02u_a2a_verbose.log | head -20
bash scripts/gpu_kernel_choices.sh
