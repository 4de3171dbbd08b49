#!/bin/bash
# round 2 evidence on the current build: full GPU suite, smoke, bench line
# (with the interposer section) + reference arm, bench launch list
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 2400 python -m pytest -q -m gpu tests > gpurun_out/r02s_pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r02s_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02s_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/r02s_bench.json 2> gpurun_out/r02s_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02s_bench_reference.json 2> gpurun_out/r02s_bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_(smallrow|words|tma|runs|batch|job|shift)' --csv --log-file gpurun_out/r02s_launches_bench.csv python bench.py --steps 1 --warmup 1 --no-halo --no-cpu-baseline > gpurun_out/r02s_ncu_bench.log 2>&1
tail -n 3 gpurun_out/r02s_pytest_gpu.log; tail -1 gpurun_out/r02s_smoke.log
python -c "
import json; d=json.load(open('gpurun_out/r02s_bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])
print(json.dumps(d.get('interpose'))[:600])"
