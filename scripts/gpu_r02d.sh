#!/bin/bash
# round 2: diagnose the send/recv hang, DRAM counters, e2e issue orders, bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
TEMPI_TIMEOUT=30 timeout 600 python -m pytest -x -q -m gpu tests/test_rt.py -k "sendrecv_every or nonblocking_pipelined or window_pressure" > gpurun_out/r02d_send.log 2>&1
echo "send rc=$?" >> gpurun_out/r02d_send.log
bash scripts/gpu_r02_counters.sh
for o in ascending interleaved descending; do
  BENCH_E2E_ORDER=$o timeout 900 python bench.py --steps 5 --warmup 3 --no-halo > gpurun_out/r02d_bench_$o.json 2> gpurun_out/r02d_bench_$o.err
done
tail -n 3 gpurun_out/r02d_send.log gpurun_out/r02_e0_counters.log
