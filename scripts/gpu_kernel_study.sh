# kernel study: the halo region / batch kernels and the typed-copy kernels against pack/unpack (cold L2)
timeout 300 python scripts/halo_regions.py 9 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print({k:(v['us'],v['GBps']) for k,v in d.items()})"
timeout 300 python scripts/copy_bench.py 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print({k:{n:x['us'] for n,x in v.items()} for k,v in d.items()})"
