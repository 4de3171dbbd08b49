timeout 600 python tools/measure_profile.py --out gpurun_out/b200.profile 2>&1 | tail -8
cp gpurun_out/b200.profile profiles/b200.profile 2>/dev/null
timeout 900 python bench.py --steps 3 --warmup 3 --cpu-seconds 3 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; tail -2 gpurun_out/bench_n1.err
python -c "import json;d=json.load(open('gpurun_out/bench_n1.json'));print(d['value'],d['halo'],d['send'])"
BENCH_BACKEND=gloo BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --incount 4 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; tail -3 gpurun_out/bench_n2.err
python -c "import json;d=json.load(open('gpurun_out/bench_n2.json'));print(d['value'],json.dumps(d['halo']),json.dumps(d['send'])[:3000])"
