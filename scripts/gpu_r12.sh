set -o pipefail
mkdir -p gpurun_out
timeout 200 python scripts/halo_sig_exp.py 2>&1 | tail -3 | tee gpurun_out/halo_sig_exp.txt
timeout 900 python bench.py 2>gpurun_out/bench.err | tee gpurun_out/bench.json
