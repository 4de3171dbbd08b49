#!/bin/bash
# round 2: stream-memory-op prologue (no in-kernel waits that need a peer's
# kernel to be resident) -- protocol tests, protocol cost, MPS multi-rank at
# 2/4/8 ranks on one GPU, latency probe old vs new, e2e with independent legs
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export TEMPI_TIMEOUT=60
timeout 1500 python -m pytest -q -m gpu tests/test_halo.py tests/test_rt.py tests/test_mpi.py tests/test_multigpu.py > gpurun_out/r02k_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r02k_pytest.log
for lib in scripts/_old/libstridepack_b200.so paper_2012_14363_b200/libstridepack_b200.so; do
  PROTO_TAG=$lib SPB_LIB=$PWD/$lib timeout 300 python scripts/protocol_cost.py 30 >> gpurun_out/r02k_protocol.jsonl 2>> gpurun_out/r02k_protocol.err
done
echo "== old" > gpurun_out/r02k_latency.txt
LD_LIBRARY_PATH=$PWD/scripts/_old timeout 300 tools/latency_probe >> gpurun_out/r02k_latency.txt 2>&1
echo "== new" >> gpurun_out/r02k_latency.txt
timeout 300 tools/latency_probe >> gpurun_out/r02k_latency.txt 2>&1
export CUDA_MPS_PIPE_DIRECTORY=/tmp/nvidia-mps CUDA_MPS_LOG_DIRECTORY=/tmp/nvidia-mps-log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d && echo "mps started" > gpurun_out/r02k_mps.txt
for n in 2 4 8; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29620+n)) \
    scripts/mps_multirank.py > gpurun_out/r02k_mps_$n.json 2> gpurun_out/r02k_mps_$n.err
  echo "n=$n rc=$?" >> gpurun_out/r02k_mps.txt
done
echo quit | nvidia-cuda-mps-control
unset CUDA_MPS_PIPE_DIRECTORY CUDA_MPS_LOG_DIRECTORY
sleep 2
for ns in 10 2; do
  BENCH_E2E_STREAMS=$ns timeout 600 python bench.py --steps 5 --warmup 3 --no-halo --no-cpu-baseline > gpurun_out/r02k_e2e_ns$ns.json 2>> gpurun_out/r02k_e2e.err
done
tail -n 3 gpurun_out/r02k_pytest.log; cat gpurun_out/r02k_mps.txt; cat gpurun_out/r02k_protocol.jsonl
