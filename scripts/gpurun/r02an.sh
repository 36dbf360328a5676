# 1 GPU: inverse + precondition parity, bench N=1, launch list (finalize share)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py --force > /dev/null
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stale.py -q -x > gpurun_out/pytest_par.log 2>&1; echo "parity tests rc=$?"; tail -1 gpurun_out/pytest_par.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-stale > gpurun_out/bench_n1.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms'])"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-stale > gpurun_out/ncu.log 2>&1; echo "ncu list rc=$?"
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/launches.csv")))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
H = rows[h]; ki = H.index("Kernel Name"); vi = H.index("Metric Value")
d = collections.defaultdict(float)
for r in rows[h + 1:]:
    if len(r) > vi: d[r[ki].split("(")[0]] += float(r[vi].replace(",", ""))
for k, v in sorted(d.items(), key=lambda x: -x[1])[:8]: print(f"{k:40s} {v/1e3/4:9.1f} us per step (4 steps incl. warmup)")
PY
