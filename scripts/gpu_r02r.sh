#!/bin/bash
# round 2: the copy-engine (DMA) path -- parity tests, then the study
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -m gpu tests/test_pack_gpu.py -k "dma or copy_engine" > gpurun_out/r02r_dma_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02r_dma_tests.log
timeout 1200 python scripts/dma_study.py --e0 512,256,128,64,32,16,8,4,2,1 --k 16 --reps 3 > gpurun_out/r02r_dma_study.jsonl 2> gpurun_out/r02r_dma_study.err
tail -n 3 gpurun_out/r02r_dma_tests.log; grep -E "FAIL|Error" gpurun_out/r02r_dma_tests.log | head; cat gpurun_out/r02r_dma_study.jsonl; tail -3 gpurun_out/r02r_dma_study.err
