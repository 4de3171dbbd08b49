#!/bin/bash
# round 2: MPI-3.1 example GPU tests, cold-L2 latency probe, default bench
# line + reference arm, bench launch list, full capture of the signalled
# DIRECT halo launch (in-kernel waits, per-CTA release counters)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python -m pytest -q -m gpu tests/test_mpi31_examples.py > gpurun_out/r02m_pytest_mpi31.log 2>&1
echo "rc=$?" >> gpurun_out/r02m_pytest_mpi31.log
timeout 300 tools/latency_probe > gpurun_out/r02m_latency.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02m_bench.json 2> gpurun_out/r02m_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02m_bench_reference.json 2> gpurun_out/r02m_bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_(smallrow|words|tma|runs|batch|job|shift)' --csv --log-file gpurun_out/r02m_launches_bench.csv python bench.py --steps 1 --warmup 1 --no-halo --no-cpu-baseline > gpurun_out/r02m_ncu_bench.log 2>&1
TEMPI_FLAG_WAIT=kernel timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_batchp --launch-skip 13 -c 1 -o gpurun_out/r02m_full_halo_direct_flags python scripts/protocol_cost.py 3 > gpurun_out/r02m_ncu_halo.log 2>&1
tail -n 2 gpurun_out/r02m_pytest_mpi31.log; cat gpurun_out/r02m_latency.txt | tail -8
