set -o pipefail
mkdir -p gpurun_out
timeout 300 python scripts/halo_regions.py 7 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print({k:(v['us'],v['GBps']) for k,v in d.items()})" | tee gpurun_out/halo_regions.txt
timeout 300 python tools/bench_parts.py 2>&1 | tail -1 | tee gpurun_out/halo_section.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_batchp -s 1 -c 1 -o gpurun_out/halo_direct5 python scripts/halo_one.py direct 3 > gpurun_out/halo_ncu.log 2>&1
timeout 1200 python -m pytest tests/test_halo.py tests/test_rt.py tests/test_mpi.py -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.log
