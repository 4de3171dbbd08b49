#!/bin/bash
# round 2: e2e with independent pack/unpack legs (stream-count variants);
# multi-rank protocol runs on one GPU under MPS (2/4/8 ranks) and without MPS
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for ns in 10 4 2; do
  BENCH_E2E_STREAMS=$ns timeout 600 python bench.py --steps 5 --warmup 3 --no-halo --no-cpu-baseline > gpurun_out/r02j_e2e_ns$ns.json 2>> gpurun_out/r02j_e2e.err
done
export TEMPI_TIMEOUT=60
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
  scripts/mps_multirank.py > gpurun_out/r02j_nomps_2.json 2> gpurun_out/r02j_nomps_2.err
export CUDA_MPS_PIPE_DIRECTORY=/tmp/nvidia-mps CUDA_MPS_LOG_DIRECTORY=/tmp/nvidia-mps-log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d && echo "mps started" > gpurun_out/r02j_mps.txt
for n in 2 4 8; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29620+n)) \
    scripts/mps_multirank.py > gpurun_out/r02j_mps_$n.json 2> gpurun_out/r02j_mps_$n.err
  echo "n=$n rc=$?" >> gpurun_out/r02j_mps.txt
done
echo quit | nvidia-cuda-mps-control
cat $CUDA_MPS_LOG_DIRECTORY/control.log >> gpurun_out/r02j_mps.txt 2>/dev/null
cat gpurun_out/r02j_mps.txt
