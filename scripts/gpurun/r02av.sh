# 1 GPU: inverse parity + bench N=1 x2 (operand load order)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -k "inverse" > gpurun_out/pytest_inv.log 2>&1; echo "inverse tests rc=$?"; tail -1 gpurun_out/pytest_inv.log
for r in 1 2; do
timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-stale --no-cpu-baseline --no-e2e > gpurun_out/bench_n1.log 2>&1
tail -1 gpurun_out/bench_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms']['inverse'])"
done
