#!/bin/bash
# round 2: MPI-4 persistent neighbour collectives (compiled typed-copy plan)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export TEMPI_TIMEOUT=60
timeout 1200 python -m pytest -q -m gpu tests/test_mpi.py -k "halo" > gpurun_out/r02ai_halo.log 2>&1
echo "rc=$?" >> gpurun_out/r02ai_halo.log
tail -n 3 gpurun_out/r02ai_halo.log; grep -E "^FAILED|FAIL rank|Error" gpurun_out/r02ai_halo.log | head
PKG=paper_2012_14363_b200
gcc -O2 -Iinclude -I/usr/local/cuda/include tests/native/mpi_halo.c -o /tmp/mpi_halo -L$PKG -ltempi_b200 -lstridepack_b200 \
  -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/$PKG
for mode in 1 2; do
  echo "mode $mode 1x1x1 256^3:"; timeout 120 python tools/tempirun.py -n 1 /tmp/mpi_halo 1 1 1 256 2 32 20 $mode | head -1
done | tee gpurun_out/r02ai_persistent_timing.txt
