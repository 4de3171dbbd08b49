#!/bin/bash
# round 2: hybrid flag waits (in-kernel when every rank has its own GPU,
# stream memory ops when ranks share one) -- full GPU suite (shared GPU:
# stream mode), protocol modules again with TEMPI_FLAG_WAIT=kernel, protocol
# cost of both modes, MPS multi-rank steady state at 1/2/4/8 ranks, e2e DMA
# chunk sweep
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export TEMPI_TIMEOUT=60
timeout 2400 python -m pytest -q -m gpu tests > gpurun_out/r02l_pytest_gpu.log 2>&1
echo "all rc=$?" >> gpurun_out/r02l_pytest_gpu.log
TEMPI_FLAG_WAIT=kernel timeout 1500 python -m pytest -q -m gpu tests/test_halo.py tests/test_rt.py tests/test_mpi.py > gpurun_out/r02l_pytest_kernelwaits.log 2>&1
echo "rc=$?" >> gpurun_out/r02l_pytest_kernelwaits.log
for mode in kernel stream; do
  PROTO_TAG=$mode TEMPI_FLAG_WAIT=$mode timeout 300 python scripts/protocol_cost.py 30 >> gpurun_out/r02l_protocol.jsonl 2>> gpurun_out/r02l_protocol.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29610 \
  scripts/mps_multirank.py > gpurun_out/r02l_mps_1.json 2> gpurun_out/r02l_mps_1.err
export CUDA_MPS_PIPE_DIRECTORY=/tmp/nvidia-mps CUDA_MPS_LOG_DIRECTORY=/tmp/nvidia-mps-log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d && echo "mps started" > gpurun_out/r02l_mps.txt
for n in 2 4 8; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29620+n)) \
    scripts/mps_multirank.py > gpurun_out/r02l_mps_$n.json 2> gpurun_out/r02l_mps_$n.err
  echo "n=$n rc=$?" >> gpurun_out/r02l_mps.txt
done
echo quit | nvidia-cuda-mps-control
unset CUDA_MPS_PIPE_DIRECTORY CUDA_MPS_LOG_DIRECTORY
sleep 2
for c in 2097152 4194304 16777216; do
  TEMPI_DMA_CHUNK=$c timeout 600 python bench.py --steps 5 --warmup 3 --no-halo --no-cpu-baseline > gpurun_out/r02l_e2e_chunk$c.json 2>> gpurun_out/r02l_e2e.err
done
tail -n 2 gpurun_out/r02l_pytest_gpu.log gpurun_out/r02l_pytest_kernelwaits.log; cat gpurun_out/r02l_mps.txt; cat gpurun_out/r02l_protocol.jsonl
