timeout 900 python -m pytest tests/test_rt.py tests/test_host_paths_gpu.py -m gpu -q 2>&1 | tail -4
timeout 900 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --incount 8 > gpurun_out/bench_async.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/bench_async.json'));print(d['halo'])"
