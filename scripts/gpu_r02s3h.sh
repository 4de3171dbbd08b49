#!/bin/bash
# bench.py's N = 2 path (the driver's scaling launch) on one B200: two ranks
# share the GPU under MPS, gloo for the bench's own reductions
# (incount 16: two ranks on one 178 GiB GPU cannot both hold 2 x 64 GiB)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export TEMPI_TIMEOUT=60
export CUDA_MPS_PIPE_DIRECTORY=/tmp/nvidia-mps CUDA_MPS_LOG_DIRECTORY=/tmp/nvidia-mps-log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d
BENCH_DEVICE=0 BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29655 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --incount 16 \
  > gpurun_out/r02s3h_bench_n2_shared.json 2> gpurun_out/r02s3h_bench_n2_shared.err
echo "rc=$?"
echo quit | nvidia-cuda-mps-control
python -c "
import json; d=json.load(open('gpurun_out/r02s3h_bench_n2_shared.json'))
print(d['n_gpus'], d['value'], d['e2e']['value'], d['halo'].get('grid'), d['halo'].get('verified'), d['halo'].get('direct_us'))
s=d.get('send'); print(json.dumps(s)[:1500])"
