# factor SYRK on the tensor-bound subset (3x3 / 7x7 convs): event time + one ncu --set full capture
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 300 python scripts/factor_subset.py tensor 10; timeout -s KILL 300 python scripts/factor_subset.py all 10
timeout -s KILL 900 ncu --set full --clock-control none -k regex:factor_syrk -c 1 -o gpurun_out/prof_factor_tensor -f python scripts/factor_subset.py tensor 1 > gpurun_out/ncu_ft.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_factor_tensor.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2]
d=dict(zip(h,v))
for k in ['gpu__time_duration.sum','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed','dram__bytes_read.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed']: print(k, d.get(k))
"
