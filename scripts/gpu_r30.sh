set -o pipefail
timeout 300 python scripts/copy_bench.py 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print({k:{n:x['us'] for n,x in v.items()} for k,v in d.items()})"
timeout 300 python tools/bench_parts.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_halo.py tests/test_pack_gpu.py tests/test_rt.py -m gpu -q -x 2>&1 | tail -2
