#!/bin/bash
# misaligned-row kernel: parity tests + throughput sweep
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_pack_gpu.py -x -q -m gpu -k "shift or corpus" 2>&1 | tail -15
timeout 300 python scripts/shift_bench.py 2>&1 | tail -120
