#!/bin/bash
# round 2: compute-sanitizer over the new kernels -- k_runs_shift (single
# packs), the copy-engine path, and k_runs_multi_shift (multi-process)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck; do
  timeout 1200 $CS --tool $tool --error-exitcode 86 --print-limit 20 python -m pytest -q -m gpu tests/test_types_ext.py -k "misaligned" \
    > gpurun_out/r02ac_${tool}_runs_shift.log 2>&1
  echo "rc=$?" >> gpurun_out/r02ac_${tool}_runs_shift.log
done
timeout 1200 $CS --tool memcheck --error-exitcode 86 --print-limit 20 python -m pytest -q -m gpu tests/test_pack_gpu.py -k "copy_engine or (corpus_parity and dma)" \
  > gpurun_out/r02ac_memcheck_dma.log 2>&1
echo "rc=$?" >> gpurun_out/r02ac_memcheck_dma.log
timeout 1200 $CS --tool memcheck --target-processes all --error-exitcode 86 --print-limit 20 python -m pytest -q -m gpu tests/test_rt.py -k "misaligned" \
  > gpurun_out/r02ac_memcheck_nbr_shift.log 2>&1
echo "rc=$?" >> gpurun_out/r02ac_memcheck_nbr_shift.log
for f in gpurun_out/r02ac_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|rc=" $f | tail -4; done
