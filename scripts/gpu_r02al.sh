#!/bin/bash
# round 2: repeat the protocol-heavy tests (graph capture, persistent plans,
# soak, alternating layouts, interposer ring) to look for intermittent failures
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
export TEMPI_TIMEOUT=60
: > gpurun_out/r02al_repeat.log
for i in $(seq 1 8); do
  timeout 600 python -m pytest -q -m gpu tests/test_rt.py -k "graph or persistent_neighbor or soak or alternating or misaligned" 2>&1 | tail -1 >> gpurun_out/r02al_repeat.log
  timeout 300 python -m pytest -q -m gpu tests/test_interpose.py -k "nonblocking_ring or device_paths" 2>&1 | tail -1 >> gpurun_out/r02al_repeat.log
done
sort gpurun_out/r02al_repeat.log | sed 's/ in [0-9.]*s.*//' | uniq -c
