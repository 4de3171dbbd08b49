#!/bin/bash
# round 2: new parity / race regression tests first, then the whole GPU suite
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt
timeout 1500 python -m pytest -x -q -m gpu tests/test_rt.py -k "irregular_receive or alternating or error_after_entry or buffer_too_small" > gpurun_out/r02a_rt_new.log 2>&1
echo "rt_new rc=$?" >> gpurun_out/r02a_rt_new.log
timeout 1200 python -m pytest -x -q -m gpu tests/test_mpi.py -k "unstructured" > gpurun_out/r02a_mpi_unstructured.log 2>&1
echo "mpi rc=$?" >> gpurun_out/r02a_mpi_unstructured.log
timeout 1500 python -m pytest -q -m gpu tests/test_pack_gpu.py -k "full_size or incount64 or tma_path" > gpurun_out/r02a_fullsize.log 2>&1
echo "full rc=$?" >> gpurun_out/r02a_fullsize.log
timeout 1800 python -m pytest -q -m gpu tests > gpurun_out/r02a_pytest_gpu.log 2>&1
echo "all rc=$?" >> gpurun_out/r02a_pytest_gpu.log
tail -3 gpurun_out/r02a_*.log
