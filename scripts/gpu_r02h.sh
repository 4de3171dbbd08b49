#!/bin/bash
# round 2 (session 2): validate HEAD -- full GPU suite, smoke, bench, reference arm
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02h_smoke.log 2>&1
timeout 2400 python -m pytest -q -m gpu tests > gpurun_out/r02h_pytest_gpu.log 2>&1
echo "all rc=$?" >> gpurun_out/r02h_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02h_bench_reference.json 2> gpurun_out/r02h_bench_reference.err
tail -n 3 gpurun_out/r02h_pytest_gpu.log; cat gpurun_out/r02h_smoke.log | tail -2
