./scripts/ldtest2 | tee gpurun_out/ldtest2.txt
ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum --clock-control none -k regex:gather --csv ./scripts/ldtest2 2>/dev/null > gpurun_out/ldtest2_ncu.csv
