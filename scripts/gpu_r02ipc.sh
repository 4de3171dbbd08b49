#!/bin/bash
# round 2: stale IPC mappings closed by base address before the open (no
# cudaErrorAlreadyMapped round trip) and DIRECT receives without a receiver
# event -- the reallocating-receiver test under memcheck, the all-to-all
# program under memcheck (the run that reported the AlreadyMapped API
# errors), the runtime / MPI / interposer suites, latency probe old vs new
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export TEMPI_TIMEOUT=300
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck --target-processes all --error-exitcode 86 --print-limit 20 \
  python -m pytest -q -m gpu -p no:cacheprovider tests/test_rt.py -k "reallocating" > gpurun_out/r02ipc_memcheck_realloc.log 2>&1
echo "rc=$?" >> gpurun_out/r02ipc_memcheck_realloc.log
timeout 900 $CS --tool memcheck --target-processes all --error-exitcode 86 --print-limit 20 \
  python -m pytest -q -m gpu -p no:cacheprovider tests/test_mpi.py -k "alltoallv_alltoallw" > gpurun_out/r02san_memcheck_alltoall.log 2>&1
echo "rc=$?" >> gpurun_out/r02san_memcheck_alltoall.log
timeout 1500 python -m pytest -q -m gpu -p no:cacheprovider tests/test_rt.py tests/test_mpi.py tests/test_interpose.py tests/test_halo.py \
  > gpurun_out/r02ipc_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r02ipc_pytest.log
for k in 1 2; do
  echo "== old $k" >> gpurun_out/r02ipc_latency.txt
  LD_LIBRARY_PATH=$PWD/scripts/_old timeout 300 tools/latency_probe >> gpurun_out/r02ipc_latency.txt 2>&1
  echo "== new $k" >> gpurun_out/r02ipc_latency.txt
  timeout 300 tools/latency_probe >> gpurun_out/r02ipc_latency.txt 2>&1
done
grep -E "ERROR SUMMARY|passed|failed|rc=" gpurun_out/r02ipc_memcheck_realloc.log gpurun_out/r02san_memcheck_alltoall.log | tail -6
tail -n 3 gpurun_out/r02ipc_pytest.log
grep -E "==|self send" gpurun_out/r02ipc_latency.txt
