# pivot band skip: inverse parity, lone-4608 chain, RN50 bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -k "inverse or step" > gpurun_out/pytest_inv.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/pytest_inv.log
timeout -s KILL 300 python scripts/one_inverse.py 4608 64
timeout -s KILL 300 python bench.py --no-cpu-baseline --no-e2e --no-stale --steps 10 > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms'])"
KFAC_NVCC_EXTRA=-DINV_TRACE python -c "import sys; sys.path.insert(0,'paper_1811_12019_b200'); import build; build.build(force=True)" > /dev/null 2>&1
timeout -s KILL 300 python scripts/trace_one.py 4608 gpurun_out/trace_one.txt > /dev/null 2>&1; echo "trace1 rc=$?"
python scripts/trace_analyze.py gpurun_out/trace_one.txt | grep "kind 5"
python paper_1811_12019_b200/build.py --force > /dev/null
