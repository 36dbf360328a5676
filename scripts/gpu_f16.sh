cd /root/repo
python paper_1811_12019_b200/build.py > /dev/null
ncu --set full --import-source on -k regex:factor_syrk -c 1 -o gpurun_out/prof_syrk -f python scripts/time_factor_all.py resnet50 > /dev/null 2>&1
ncu -i gpurun_out/prof_syrk.ncu-rep --page raw --csv 2>/dev/null > gpurun_out/prof_syrk_raw.csv
python - <<'PY'
import csv
r=list(csv.reader(open('gpurun_out/prof_syrk_raw.csv'))); h=r[0]; v=r[2]
want=['gpu__time_duration.sum','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed','sm__cycles_active.avg','smsp__cycles_active.avg','gpc__cycles_elapsed.max','sm__throughput.avg.pct_of_peak_sustained_elapsed','dram__bytes_read.sum','dram__bytes_write.sum','l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum','lts__t_sectors_srcunit_tex_op_read.sum','smsp__inst_executed.sum','sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active']
for k in want:
    if k in h: print(k, v[h.index(k)])
for i,k in enumerate(h):
    if 'pipe_tensor' in k or ('clock' in k.lower() and 'sm' in k.lower()): print(k, v[i])
PY
