# 1 GPU: final default bench line at HEAD (every key)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 900 python bench.py > gpurun_out/bench_n1.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
