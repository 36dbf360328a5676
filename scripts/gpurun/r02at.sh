# 1 GPU: smoke + parity subset + bench with the NVTX ranges
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wire.py tests/test_gpu_stale.py -q -x > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_q.log
timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-stale --no-cpu-baseline > gpurun_out/bench_n1.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms'])"
