#!/bin/bash
# bench.py's N = 4 and 8 launches on one B200 (ranks share the GPU under
# MPS; incount scaled down so every rank's buffers fit one 178 GiB GPU)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export TEMPI_TIMEOUT=60
export CUDA_MPS_PIPE_DIRECTORY=/tmp/nvidia-mps CUDA_MPS_LOG_DIRECTORY=/tmp/nvidia-mps-log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d
for n in 4 8; do
  k=$((32 / n))
  BENCH_DEVICE=0 BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29660 + n)) bench.py --gpus $n --steps 3 --warmup 3 --no-cpu-baseline \
    --incount $k --e2e-incount $k > gpurun_out/r02s3i_bench_n${n}_shared.json 2> gpurun_out/r02s3i_bench_n${n}_shared.err
  echo "n=$n rc=$?"
done
echo quit | nvidia-cuda-mps-control
for n in 4 8; do python -c "
import json; d=json.load(open('gpurun_out/r02s3i_bench_n${n}_shared.json'))
h=d['halo']; s=d.get('send') or {}
print(d['n_gpus'], d['value'], h.get('grid'), h.get('verified'), h.get('direct_us'), h.get('mpi_alltoallw_us'), (s.get('checks') if isinstance(s, dict) else s))" 2>&1 | tail -2; done
