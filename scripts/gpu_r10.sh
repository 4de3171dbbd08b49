set -o pipefail
mkdir -p gpurun_out
timeout 300 python tools/bench_parts.py 2>&1 | tail -1 | tee gpurun_out/halo_section.json
timeout 300 python scripts/halo_regions.py 7 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print({k:(v['us'],v['GBps']) for k,v in d.items()})" | tee gpurun_out/halo_regions.txt
