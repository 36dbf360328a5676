# inverse parity tests + RN50 bench + lone-4608 trace (INV_TRACE build)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 600 python -m pytest tests -q -m gpu -s -p no:cacheprovider -k "inverse or step" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAIL|Error" gpurun_out/pytest_gpu.log | tail -3
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms'])"
timeout -s KILL 120 python scripts/one_inverse.py 4608 512 2>&1 | tail -1
KFAC_NVCC_EXTRA=-DINV_TRACE python -c "import sys; sys.path.insert(0,'paper_1811_12019_b200'); import build; build.build(force=True)" > /dev/null 2>&1
timeout -s KILL 300 python scripts/trace_one.py 4608 gpurun_out/trace_one.txt; echo "trace rc=$?"
python scripts/trace_analyze.py gpurun_out/trace_one.txt | tail -9
timeout -s KILL 300 python scripts/trace_step.py gpurun_out/trace_step.txt > /dev/null; python scripts/trace_analyze.py gpurun_out/trace_step.txt | tail -9
