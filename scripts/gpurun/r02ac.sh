# 1 GPU: inverse parity + bench N=1 + fullsize RN50 (both gammas)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -k "inverse" > gpurun_out/pytest_inv.log 2>&1; echo "inverse tests rc=$?"; tail -3 gpurun_out/pytest_inv.log
timeout -s KILL 600 python bench.py > gpurun_out/bench_n1.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms'], d['e2e']['value'], d['clocks'])"
timeout -s KILL 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -s -k "resnet50" > gpurun_out/pytest_full.log 2>&1; echo "fullsize rc=$?"; grep -E "worst|passed|failed" gpurun_out/pytest_full.log | tail -3
