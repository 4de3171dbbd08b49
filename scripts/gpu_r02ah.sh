#!/bin/bash
# round 2: graph-captured distributed halo exchanges under MPS (ranks truly
# concurrent on one GPU, stream flag-wait mode with the one-warp wait kernel)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export TEMPI_TIMEOUT=60
export CUDA_MPS_PIPE_DIRECTORY=/tmp/nvidia-mps CUDA_MPS_LOG_DIRECTORY=/tmp/nvidia-mps-log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d && echo "mps started" > gpurun_out/r02ah_mps_graph.log
timeout 900 python -m pytest -q -m gpu tests/test_rt.py -k "graph or soak" >> gpurun_out/r02ah_mps_graph.log 2>&1
echo "rc=$?" >> gpurun_out/r02ah_mps_graph.log
echo quit | nvidia-cuda-mps-control
tail -n 4 gpurun_out/r02ah_mps_graph.log
