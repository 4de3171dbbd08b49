#!/bin/bash
# bench twice back to back (clock sampler check) + the reference arm
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for i in 1 2; do
  timeout 1200 python bench.py > gpurun_out/r02s3c_bench_$i.json 2> gpurun_out/r02s3c_bench_$i.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02s3c_bench_reference.json 2> gpurun_out/r02s3c_bench_reference.err
for i in 1 2; do python -c "
import json; d=json.load(open('gpurun_out/r02s3c_bench_$i.json')); print(d['value'], d['e2e']['value'], d['clocks'])"; done
python -c "import json; r=json.load(open('gpurun_out/r02s3c_bench_reference.json')); print('reference', r.get('value'), r.get('config'))"
