set -o pipefail
mkdir -p gpurun_out
timeout 200 python scripts/halo_sig_exp.py 2>&1 | tail -3 | tee gpurun_out/halo_sig_exp.txt
timeout 300 python scripts/e2e_exp.py 2>&1 | tail -40 | tee gpurun_out/e2e_exp.txt
