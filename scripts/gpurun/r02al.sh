# 1 GPU: parity + bench + pivot phases
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py --force > /dev/null
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -k "inverse" > gpurun_out/pytest_inv.log 2>&1; echo "inverse tests rc=$?"; tail -1 gpurun_out/pytest_inv.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-stale > gpurun_out/bench_n1.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms'])"
KFAC_NVCC_EXTRA="-DPIVOT_DBG" python paper_1811_12019_b200/build.py --force > /dev/null 2>&1
timeout -s KILL 300 python scripts/pivot_phases.py > gpurun_out/pivot_phases.txt 2>&1; head -3 gpurun_out/pivot_phases.txt; grep sweep gpurun_out/pivot_phases.txt
