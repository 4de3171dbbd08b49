set -o pipefail
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.log
timeout 900 python bench.py 2>gpurun_out/bench.err | tee gpurun_out/bench.json
