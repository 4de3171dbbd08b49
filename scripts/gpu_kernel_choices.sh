#!/bin/bash
# ncu counters for every automatic kernel choice (scripts/kernel_choices.py)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,lts__t_requests_srcunit_tex.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed
timeout 1500 ncu --metrics $M --clock-control none -k regex:'k_(smallrow|words|tma|runs|batch|job|shift)' --csv --log-file gpurun_out/r02_kernel_choices.csv python scripts/kernel_choices.py > gpurun_out/r02_kernel_choices.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r02_kernel_choices.log
python scripts/kernel_choices_table.py gpurun_out/r02_kernel_choices.csv gpurun_out/r02_kernel_choices.log gpurun_out/r02_kernel_choices.md > gpurun_out/r02_kernel_choices_table.err 2>&1
cat gpurun_out/r02_kernel_choices.md; tail -3 gpurun_out/r02_kernel_choices_table.err; tail -3 gpurun_out/r02_kernel_choices.log
