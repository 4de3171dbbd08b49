#!/bin/bash
# round 2: k_runs_shift -- parity, misaligned-runs study, kernel-choice counters
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_types_ext.py tests/test_pack_gpu.py -k "misaligned or random_descriptions or irregular or corpus_parity or unsupported" > gpurun_out/r02w_runs_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02w_runs_tests.log
tail -n 3 gpurun_out/r02w_runs_tests.log
timeout 900 python scripts/runs_bench.py --misaligned > gpurun_out/r02w_runs_misaligned.jsonl 2> gpurun_out/r02w_runs_misaligned.err
cat gpurun_out/r02w_runs_misaligned.jsonl; tail -3 gpurun_out/r02w_runs_misaligned.err
bash scripts/gpu_kernel_choices.sh | tail -8
