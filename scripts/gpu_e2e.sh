timeout 600 python -m pytest tests/test_host_paths_gpu.py tests/test_pack_gpu.py tests/test_rt.py -m gpu -q 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 2 --no-halo --no-cpu-baseline > gpurun_out/bench_e2e.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/bench_e2e.json'));print(d['value'],d['e2e'])"
