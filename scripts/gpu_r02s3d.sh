#!/bin/bash
# 256-bit vs 128-bit accesses on cfg2 rows (scripts/wide_access.cu)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 ./scripts/wide_access 64 > gpurun_out/r02s3f_wide_access.jsonl 2>&1
cat gpurun_out/r02s3f_wide_access.jsonl
