#!/bin/bash
# round 2: interposer over the stand-in system MPI -- GPU tests and the
# with/without-interposer timing section
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_interpose.py > gpurun_out/r02o_interpose.log 2>&1
echo "rc=$?" >> gpurun_out/r02o_interpose.log
timeout 400 python -c "
import json, sys; sys.path.insert(0, '.')
from tools.bench_parts import interpose_section
print(json.dumps(interpose_section(), indent=1))" > gpurun_out/r02o_interpose_section.json 2> gpurun_out/r02o_interpose_section.err
tail -n 3 gpurun_out/r02o_interpose.log; cat gpurun_out/r02o_interpose_section.json; tail -5 gpurun_out/r02o_interpose_section.err
