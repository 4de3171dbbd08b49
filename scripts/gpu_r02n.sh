#!/bin/bash
# round 2 (re-entry): full GPU suite, smoke, default bench line + reference arm on HEAD
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r02n_gpus.txt 2>&1
timeout 1500 python -m pytest -q -m gpu tests > gpurun_out/r02n_pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r02n_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02n_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02n_bench_reference.json 2> gpurun_out/r02n_bench_reference.err
tail -n 3 gpurun_out/r02n_pytest_gpu.log; cat gpurun_out/r02n_smoke.log | tail -2
