cd /root/repo
python paper_1811_12019_b200/build.py > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/factor_launches.csv python scripts/time_factor_all.py resnet50 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/factor_launches.csv')))
h=None
for i,r in enumerate(rows):
    if 'Kernel Name' in r: h=r; start=i+1; break
ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
for r in rows[start:start+40]:
    print(r[ki][:40], r[vi], r[ui])
PY
