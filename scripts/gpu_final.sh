# full round-end style run: tests, smoke, bench (+ reference arm), launch list, TMA E0=64 capture
set -o pipefail
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.log
timeout 900 python bench.py 2>gpurun_out/bench.err | tee gpurun_out/bench.json
timeout 600 python bench.py --impl reference 2>gpurun_out/bench_ref.err | tee gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 0 --no-halo > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tma -c 1 -o gpurun_out/r01_full_unpack_e0_64_tma python scripts/prof_cfg2.py --e0 64 --k 64 --reps 1 --mode unpack > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep | tail -2
