#!/bin/bash
# round 2: k_runs_multi_shift -- misaligned irregular neighbour edges, the
# other irregular/neighbour tests, the single-pack shift tests
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -m gpu tests/test_rt.py tests/test_types_ext.py tests/test_mpi.py -k "irregular or misaligned or unstructured or neighbor or random_descriptions" > gpurun_out/r02ab_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02ab_tests.log
tail -n 4 gpurun_out/r02ab_tests.log; grep -E "^FAILED|Error" gpurun_out/r02ab_tests.log | head
