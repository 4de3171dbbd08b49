#!/bin/bash
# round 2: blocking (legacy-ordered) streams for the MPI-facing work; set
# completions; full GPU suite + bench line
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 2400 python -m pytest -q -m gpu tests > gpurun_out/r02z_pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r02z_pytest_gpu.log
tail -n 4 gpurun_out/r02z_pytest_gpu.log; grep -E "^FAILED" gpurun_out/r02z_pytest_gpu.log | head
timeout 1200 python bench.py > gpurun_out/r02z_bench.json 2> gpurun_out/r02z_bench.err
python -c "
import json; d=json.load(open('gpurun_out/r02z_bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['halo']['direct_us'], d['send']['checks'])"
