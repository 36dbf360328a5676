# 1 GPU: inverse parity + bench N=1 + trace summary
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
KFAC_NVCC_EXTRA="$EXTRA" python paper_1811_12019_b200/build.py --force > /dev/null
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -k "inverse" > gpurun_out/pytest_inv.log 2>&1; echo "inverse tests rc=$?"; tail -2 gpurun_out/pytest_inv.log
timeout -s KILL 600 python bench.py > gpurun_out/bench_n1.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms'], d['e2e']['value'], d['clocks'])"
KFAC_NVCC_EXTRA="-DINV_TRACE $EXTRA" python paper_1811_12019_b200/build.py --force > /dev/null 2>&1
timeout -s KILL 600 python scripts/trace_step.py gpurun_out/trace.txt > gpurun_out/trace_run.log 2>&1; echo "trace rc=$?"
python scripts/trace_analyze.py gpurun_out/trace.txt > gpurun_out/trace_summary.txt 2>&1; grep -E "kind|total" gpurun_out/trace_summary.txt
