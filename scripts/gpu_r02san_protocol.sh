#!/bin/bash
# round 2: compute-sanitizer over the protocol pieces added this round --
# halo plans captured into CUDA graphs (tick kernel, one-warp pre-wait
# kernel, device-numbered flags), MPI-4 persistent neighbour plans (eager and
# replayed), MPI_Alltoallv/w with derived types, and the interposer in front
# of the stand-in MPI. Multi-process cases use --target-processes all.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
export TEMPI_TIMEOUT=600
run() { # name tool filter...
  local name=$1 tool=$2
  shift 2
  timeout 1500 $CS --tool $tool --target-processes all --error-exitcode 86 --print-limit 20 \
    python -m pytest -q -m gpu -p no:cacheprovider "$@" > gpurun_out/r02san_${tool}_${name}.log 2>&1
  echo "rc=$?" >> gpurun_out/r02san_${tool}_${name}.log
}
for tool in memcheck racecheck synccheck; do
  run graph_one_rank $tool tests/test_halo.py -k "graph_capture_one_rank"
done
run graph_2ranks memcheck "tests/test_rt.py::test_distributed_halo_graph_capture[ranks0-3]" \
  "tests/test_rt.py::test_distributed_halo_graph_capture[ranks1-2]"
run graph_stream memcheck tests/test_rt.py -k "graph_capture_stream_mode"
run persistent memcheck tests/test_rt.py -k "persistent_neighbor_plan"
run alltoall memcheck tests/test_mpi.py -k "alltoallv_alltoallw"
run mpi_halo_persistent memcheck "tests/test_mpi.py::test_mpi_halo_exchange[grid0-2]" \
  "tests/test_mpi.py::test_mpi_halo_exchange[grid0-3]" "tests/test_mpi.py::test_mpi_halo_exchange[grid1-2]" \
  "tests/test_mpi.py::test_mpi_halo_exchange[grid1-3]"
run interposed_a2a memcheck tests/test_interpose.py -k "interposed_alltoall"
run interposed_halo memcheck "tests/test_interpose.py::test_interposed_halo_exchange[grid1-1]" \
  "tests/test_interpose.py::test_interposed_halo_exchange[grid1-2]"
for f in gpurun_out/r02san_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" $f | tail -4; done
