# prologue/epilogue flattening + side-stream task list: inverse parity, bench, launch list
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stale.py -x -q > gpurun_out/pytest_inv.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/pytest_inv.log
timeout -s KILL 300 python bench.py --no-cpu-baseline --no-e2e --no-stale --steps 10 > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms'])"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_t.csv python scripts/step_once.py resnet50 1 > /dev/null 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launches_t.csv')))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]; h=rows[hi]
k=h.index('Kernel Name'); v=h.index('Metric Value'); u=h.index('Metric Unit')
agg={}
for r in rows[hi+1:]:
    if len(r)>v:
        x=float(r[v].replace(',','')); x*= {'ns':1e-3,'us':1,'ms':1e3}.get(r[u],1)
        n=r[k].split('(')[0].split('::')[-1]; agg[n]=agg.get(n,0)+x
for n,x in sorted(agg.items(), key=lambda t:-t[1]): print(f"{n:32s} {x:9.1f} us")
PY
