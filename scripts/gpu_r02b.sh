#!/bin/bash
# round 2: re-run the neighbour-protocol regressions after the version-snapshot fix
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
free -g > gpurun_out/r02b_free.txt; nproc >> gpurun_out/r02b_free.txt
timeout 1500 python -m pytest -x -q -m gpu tests/test_rt.py -k "alternating or error_after_entry or buffer_too_small or times_out or irregular or layout_changes or nbrv or alltoallv" > gpurun_out/r02b_rt.log 2>&1
echo "rt rc=$?" >> gpurun_out/r02b_rt.log
timeout 900 python -m pytest -x -q -m gpu tests/test_pack_gpu.py -k "full_size_vs_oracle" > gpurun_out/r02b_full.log 2>&1
echo "full rc=$?" >> gpurun_out/r02b_full.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
echo "bench rc=$?" >> gpurun_out/r02b_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02b_bench_ref.json 2> gpurun_out/r02b_bench_ref.err
echo "ref rc=$?" >> gpurun_out/r02b_bench_ref.err
for f in gpurun_out/r02b_rt.log gpurun_out/r02b_full.log; do tail -n 3 $f; done
