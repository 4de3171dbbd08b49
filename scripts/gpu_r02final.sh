#!/bin/bash
# round 2 final evidence on the final build: full GPU suite, smoke, bench
# line (+ interposer section) and the reference arm, the bench launch list,
# every automatic kernel choice under ncu, and a full capture of the
# dominant kernel (cfg2 E0 = 1 unpack) and of the new shift run kernel
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r02final_gpus.txt 2>&1
timeout 2400 python -m pytest -q -m gpu tests > gpurun_out/r02final_pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r02final_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02final_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/r02final_bench.json 2> gpurun_out/r02final_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02final_bench_reference.json 2> gpurun_out/r02final_bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_(smallrow|words|tma|runs|batch|job|shift)' --csv --log-file gpurun_out/r02final_launches_bench.csv python bench.py --steps 1 --warmup 1 --no-halo --no-cpu-baseline > gpurun_out/r02final_ncu_bench.log 2>&1
bash scripts/gpu_kernel_choices.sh > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_smallrow<1, 0>|k_runs_shift' -c 3 -o gpurun_out/r02final_full_e0_1_and_shift python scripts/kernel_choices.py > gpurun_out/r02final_ncu_full.log 2>&1
tail -n 3 gpurun_out/r02final_pytest_gpu.log; tail -1 gpurun_out/r02final_smoke.log
python -c "
import json; d=json.load(open('gpurun_out/r02final_bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'], d['halo']['direct_us'])
r=json.load(open('gpurun_out/r02final_bench_reference.json')); print('reference', r.get('value'))"
