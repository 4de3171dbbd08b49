#!/bin/bash
# round 2: the runtime's in-kernel flag waits (the distinct-GPU mode) and the
# MPS multi-rank steady state on the current build (blocking streams, stale
# IPC eviction)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export TEMPI_TIMEOUT=60
TEMPI_FLAG_WAIT=kernel timeout 1500 python -m pytest -q -m gpu tests/test_halo.py tests/test_rt.py tests/test_mpi.py > gpurun_out/r02aa_pytest_kernelwaits.log 2>&1
echo "rc=$?" >> gpurun_out/r02aa_pytest_kernelwaits.log
tail -n 3 gpurun_out/r02aa_pytest_kernelwaits.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29610 \
  scripts/mps_multirank.py > gpurun_out/r02aa_mps_1.json 2> gpurun_out/r02aa_mps_1.err
export CUDA_MPS_PIPE_DIRECTORY=/tmp/nvidia-mps CUDA_MPS_LOG_DIRECTORY=/tmp/nvidia-mps-log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d && echo "mps started" > gpurun_out/r02aa_mps.txt
for n in 2 4 8; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29620+n)) \
    scripts/mps_multirank.py > gpurun_out/r02aa_mps_$n.json 2> gpurun_out/r02aa_mps_$n.err
  echo "n=$n rc=$?" >> gpurun_out/r02aa_mps.txt
done
echo quit | nvidia-cuda-mps-control
cat gpurun_out/r02aa_mps.txt
for n in 1 2 4 8; do python -c "
import json,sys
d=json.load(open('gpurun_out/r02aa_mps_$n.json'))
print($n, d['direct'], d['fused_async'], d['alltoallw'])" 2>&1 | tail -1; done
