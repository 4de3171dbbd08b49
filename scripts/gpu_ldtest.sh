./scripts/ldtest
ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum --clock-control none -k regex:gather8 --csv ./scripts/ldtest 2>/dev/null | grep -v "^==" > gpurun_out/ldtest_ncu.csv
python3 - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/ldtest_ncu.csv')))
h=rows[0]
for r in rows[1:]:
    d=dict(zip(h,r))
    if 'Kernel Name' in d: print(d['Kernel Name'][:22], d['Metric Name'], d['Metric Value'])
PY
