cd /root/repo
python paper_1811_12019_b200/build.py > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/step_launches.csv python scripts/step_once.py resnet50 1 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/step_launches.csv')))
for i,r in enumerate(rows):
    if 'Kernel Name' in r: h=r; start=i+1; break
ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
tot=collections.OrderedDict(); cnt=collections.Counter()
for r in rows[start:]:
    name=r[ki].split('(')[0].replace('void ','').replace('kfac::','')
    v=float(r[vi].replace(',',''))*(1e-3 if r[ui]=='ns' else (1 if r[ui]=='us' else 1e3))
    tot[name]=tot.get(name,0)+v; cnt[name]+=1
for k,v in sorted(tot.items(), key=lambda x:-x[1])[:20]: print(f"{k:40s} {cnt[k]:5d} {v:10.1f} us")
PY
