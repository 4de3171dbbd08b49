#!/bin/bash
# round 2: neighbour regression, B200 profile with the DIRECT surface, full GPU suite
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_rt.py -k "alternating" > gpurun_out/r02c_alt.log 2>&1
echo "alt rc=$?" >> gpurun_out/r02c_alt.log
timeout 900 ./tools/measure_profile gpurun_out/b200.profile 25 > gpurun_out/r02c_measure.txt 2>&1
echo "measure rc=$?" >> gpurun_out/r02c_measure.txt
cp gpurun_out/b200.profile profiles/b200.profile 2>/dev/null
timeout 2400 python -m pytest -q -m gpu tests > gpurun_out/r02c_pytest_gpu.log 2>&1
echo "all rc=$?" >> gpurun_out/r02c_pytest_gpu.log
tail -n 3 gpurun_out/r02c_alt.log gpurun_out/r02c_pytest_gpu.log
