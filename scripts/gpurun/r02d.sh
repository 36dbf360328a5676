# int8-sliced (Ozaki) inverse updates: parity of the inverse tests in both modes, full-size step parity, bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -s -k "inverse" > gpurun_out/pytest_inv.log 2>&1; echo "inv rc=$?"; grep -E "err|passed|failed|Error" gpurun_out/pytest_inv.log | tail -30
timeout -s KILL 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_resnet50.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_resnet50.log | cut -c1-700
timeout -s KILL 1800 python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/pytest_fullsize.log 2>&1; echo "fullsize rc=$?"; grep -E "worst|passed|failed|Error" gpurun_out/pytest_fullsize.log | tail -12
