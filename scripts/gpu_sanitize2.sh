# racecheck / synccheck on the shared-memory kernels (TMA ring, batch job
# staging), memcheck across processes on the runtime paths
set -o pipefail
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck synccheck; do
  timeout 900 $CS --tool $tool --error-exitcode 86 --print-limit 20 python -m pytest -q -x -m gpu \
    tests/test_pack_gpu.py -k "tma_path or tma_cfg2" 2>&1 | tail -4 | tee gpurun_out/${tool}_tma.log
  timeout 900 $CS --tool $tool --error-exitcode 86 --print-limit 20 python -m pytest -q -x -m gpu \
    tests/test_halo.py -k "batch_parity or copy_batch" 2>&1 | tail -4 | tee gpurun_out/${tool}_batch.log
done
timeout 1200 $CS --tool memcheck --target-processes all --error-exitcode 86 --print-limit 20 python -m pytest -q -x -m gpu \
  tests/test_rt.py -k "nonblocking or sendrecv or distributed_halo" 2>&1 | tail -4 | tee gpurun_out/memcheck_rt.log
timeout 1200 $CS --tool memcheck --target-processes all --error-exitcode 86 --print-limit 20 python -m pytest -q -x -m gpu \
  tests/test_rt.py -k "irregular or layout or alltoallv" 2>&1 | tail -5 | tee gpurun_out/memcheck_rt_irregular.log
