# round-end style verification on one B200: GPU tests, smoke, bench, reference arm
# Full verification on one B200: GPU tests, smoke, default bench, reference arm.
set -o pipefail
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv | tee gpurun_out/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee gpurun_out/smoke.log
timeout 900 python bench.py 2>gpurun_out/bench.err | tee gpurun_out/bench.json
timeout 900 python bench.py --impl reference 2>gpurun_out/bench_ref.err | tee gpurun_out/bench_ref.json
