#!/bin/bash
# DRAM / L2 counters of the E0 = 32..512 pack and unpack kernels (K = 64)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__sectors_read.sum,dram__sectors_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,dram__cycles_active.avg.pct_of_peak_sustained_elapsed,dram__cycles_active_read.avg.pct_of_peak_sustained_elapsed,dram__cycles_active_write.avg.pct_of_peak_sustained_elapsed,fbpa__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__d_sectors_fill_device.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed
timeout 900 ncu --metrics $M --clock-control none -k regex:'k_words|k_tma|k_smallrow|copy|elementwise' --csv --log-file gpurun_out/r02_e0_counters.csv python scripts/e0_counters.py > gpurun_out/r02_e0_counters.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r02_e0_counters.log
