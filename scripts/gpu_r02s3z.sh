#!/bin/bash
# session-3 last commit: full GPU suite, smoke, bench: full GPU suite, smoke, bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 2400 python -m pytest -q -m gpu tests > gpurun_out/r02s3z_pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r02s3z_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02s3z_smoke.log 2>&1
timeout 1200 python bench.py > gpurun_out/r02s3z_bench.json 2> gpurun_out/r02s3z_bench.err
tail -n 3 gpurun_out/r02s3z_pytest_gpu.log; tail -1 gpurun_out/r02s3z_smoke.log
python -c "
import json; d=json.load(open('gpurun_out/r02s3z_bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
