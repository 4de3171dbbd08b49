#!/bin/bash
# round 2: k_runs_shift v2 (one aligned load per written block, neighbour's by shuffle)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_types_ext.py tests/test_pack_gpu.py -k "misaligned or random_descriptions or irregular or corpus_parity or unsupported" > gpurun_out/r02x_runs_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02x_runs_tests.log
tail -n 3 gpurun_out/r02x_runs_tests.log
timeout 900 python scripts/runs_bench.py --misaligned > gpurun_out/r02x_runs_misaligned.jsonl 2> gpurun_out/r02x_runs_misaligned.err
python -c "
import json
for l in open('gpurun_out/r02x_runs_misaligned.jsonl'):
    r = json.loads(l); print(r['mean_block'], r['auto_word'], r['auto_pack_GBps'], r['plain_pack_GBps'], r['auto_unpack_GBps'], r['plain_unpack_GBps'])
"; tail -3 gpurun_out/r02x_runs_misaligned.err
