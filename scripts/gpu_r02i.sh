#!/bin/bash
# round 2: per-CTA release counters -- protocol parity tests, protocol cost
# old vs new, e2e issue orders with the chunked DMA pipeline
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
which nvidia-cuda-mps-control nvidia-smi > gpurun_out/r02i_tools.txt 2>&1
timeout 1500 python -m pytest -q -m gpu tests/test_halo.py tests/test_rt.py tests/test_mpi.py tests/test_multigpu.py > gpurun_out/r02i_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r02i_pytest.log
for lib in scripts/_old/libstridepack_b200.so paper_2012_14363_b200/libstridepack_b200.so; do
  PROTO_TAG=$lib SPB_LIB=$PWD/$lib timeout 300 python scripts/protocol_cost.py 30 >> gpurun_out/r02i_protocol.jsonl 2>> gpurun_out/r02i_protocol.err
done
for o in ascending pipelined descending interleaved; do
  BENCH_E2E_ORDER=$o timeout 600 python bench.py --steps 5 --warmup 3 --no-halo --no-cpu-baseline > gpurun_out/r02i_order_$o.json 2>> gpurun_out/r02i_orders.err
done
tail -n 3 gpurun_out/r02i_pytest.log; cat gpurun_out/r02i_protocol.jsonl
