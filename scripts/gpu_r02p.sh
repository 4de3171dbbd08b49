#!/bin/bash
# round 2: interposer tests + the with/without-interposer section (halo
# cases added, contiguous fast path in the stand-in MPI), then the
# compute-sanitizer pass over the irregular-receive program and the
# alternating-layout neighbour regression (scripts/gpu_sanitize_r02.sh)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_interpose.py > gpurun_out/r02p_interpose.log 2>&1
echo "rc=$?" >> gpurun_out/r02p_interpose.log
timeout 600 python -c "
import json, sys; sys.path.insert(0, '.')
from tools.bench_parts import interpose_section
print(json.dumps(interpose_section(), indent=1))" > gpurun_out/r02p_interpose_section.json 2> gpurun_out/r02p_interpose_section.err
tail -n 3 gpurun_out/r02p_interpose.log; cat gpurun_out/r02p_interpose_section.json; tail -5 gpurun_out/r02p_interpose_section.err
bash scripts/gpu_sanitize_r02.sh
