#!/bin/bash
# flakiness check: the full GPU suite twice more on the final build
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for i in 1 2; do
  timeout 1500 python -m pytest -q -m gpu tests -p no:cacheprovider > gpurun_out/r02s3g_pytest_gpu_$i.log 2>&1
  echo "rc=$?" >> gpurun_out/r02s3g_pytest_gpu_$i.log
  tail -n 2 gpurun_out/r02s3g_pytest_gpu_$i.log
done
