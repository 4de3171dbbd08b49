# bench + launch list of the same command (B200_PROFILING.md)
TAG=${TAG:-r01}
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-incount 1 > gpurun_out/bench_ncu_$TAG.log 2>&1
tail -2 gpurun_out/bench_ncu_$TAG.log
