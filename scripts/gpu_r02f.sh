#!/bin/bash
# round 2: full GPU suite, bench + reference arm, launch list, cfg1 full captures
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 2400 python -m pytest -q -m gpu tests > gpurun_out/r02f_pytest_gpu.log 2>&1
echo "all rc=$?" >> gpurun_out/r02f_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02f_bench_reference.json 2> gpurun_out/r02f_bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_(smallrow|words|tma|runs|batch|job|shift)' --csv --log-file gpurun_out/r02f_launches_bench.csv python bench.py --steps 1 --warmup 1 --no-halo --no-cpu-baseline > gpurun_out/r02f_ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_smallrow' -o gpurun_out/r02_full_cfg1 python scripts/cfg1_kernels.py > gpurun_out/r02f_ncu_cfg1.log 2>&1
tail -n 2 gpurun_out/r02f_pytest_gpu.log
