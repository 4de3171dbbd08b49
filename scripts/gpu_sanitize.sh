# compute-sanitizer memcheck over the kernel-parity tests (every kernel
# family on the golden corpus, misaligned rows, batches, typed copies)
set -o pipefail
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --error-exitcode 86 --print-limit 20 python -m pytest -q -x -m gpu \
  tests/test_pack_gpu.py -k "kat or corpus_parity or shift or smallrow or tma_path or pinned" 2>&1 | tail -25 | tee gpurun_out/sanitize_pack.log
timeout 900 $CS --tool memcheck --error-exitcode 86 --print-limit 20 python -m pytest -q -x -m gpu \
  tests/test_halo.py -k "batch or copy or randomized" 2>&1 | tail -25 | tee gpurun_out/sanitize_halo.log
timeout 900 $CS --tool memcheck --error-exitcode 86 --print-limit 20 python -m pytest -q -x -m gpu \
  tests/test_types_ext.py 2>&1 | tail -25 | tee gpurun_out/sanitize_types.log
