#!/bin/bash
# round 2: graph-capturable halo exchanges (device-numbered iterations)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export TEMPI_TIMEOUT=60
timeout 1500 python -m pytest -q -m gpu tests/test_halo.py tests/test_rt.py -k "graph or halo" > gpurun_out/r02ae_graph.log 2>&1
echo "rc=$?" >> gpurun_out/r02ae_graph.log
tail -n 4 gpurun_out/r02ae_graph.log; grep -E "^FAILED|Error|assert" gpurun_out/r02ae_graph.log | head
