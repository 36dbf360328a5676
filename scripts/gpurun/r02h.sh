# trace + quick bench of the inverse
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
KFAC_NVCC_EXTRA=-DINV_TRACE python -c "import sys; sys.path.insert(0,'paper_1811_12019_b200'); import build; build.build(force=True)" > /dev/null 2>&1
timeout -s KILL 300 python scripts/trace_step.py gpurun_out/trace_step.txt > gpurun_out/trace.log 2>&1; echo "trace rc=$?"
python scripts/trace_analyze.py gpurun_out/trace_step.txt | grep -v "^ *[0-9]" | tail -12; grep -A10 "int8 update" gpurun_out/trace.log
python paper_1811_12019_b200/build.py --force > /dev/null
timeout -s KILL 300 python scripts/one_inverse.py 4608 64
timeout -s KILL 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_resnet50.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_resnet50.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms'])"
