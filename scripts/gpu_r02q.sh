#!/bin/bash
# round 2: every interposer GPU test (incl. the unmodified engine programs
# over the stand-in system MPI) and the with/without-interposer section
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -m gpu tests/test_interpose.py > gpurun_out/r02q_interpose.log 2>&1
echo "rc=$?" >> gpurun_out/r02q_interpose.log
timeout 900 python -c "
import json, sys, time; sys.path.insert(0, '.')
from tools.bench_parts import interpose_section
t = time.time(); r = interpose_section(); r['section_s'] = round(time.time() - t, 1)
print(json.dumps(r, indent=1))" > gpurun_out/r02q_interpose_section.json 2> gpurun_out/r02q_interpose_section.err
tail -n 3 gpurun_out/r02q_interpose.log; cat gpurun_out/r02q_interpose_section.json; tail -5 gpurun_out/r02q_interpose_section.err
