#!/bin/bash
# round 2: bench launch list (ncu), e2e issue orders
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_(smallrow|words|tma|runs|batch|job|shift)' --csv --log-file gpurun_out/r02g_launches_bench.csv python bench.py --steps 1 --warmup 1 --no-halo --no-cpu-baseline > gpurun_out/r02g_ncu_bench.log 2>&1
for o in pipelined descending pipelined descending; do
  BENCH_E2E_ORDER=$o timeout 900 python bench.py --steps 5 --warmup 3 --no-halo --no-cpu-baseline >> gpurun_out/r02g_orders.jsonl 2>> gpurun_out/r02g_orders.err
done
