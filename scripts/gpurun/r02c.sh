# precond accuracy: RN tf32 split + segmented TMEM accumulation; full-size step parity + all GPU tests
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 2400 python -m pytest tests/test_gpu_fullsize.py -q -s > gpurun_out/pytest_fullsize.log 2>&1; echo "fullsize rc=$?"; grep -E "worst|passed|failed|Error" gpurun_out/pytest_fullsize.log | tail -12
timeout -s KILL 1200 python -m pytest tests -q -m gpu --deselect tests/test_gpu_fullsize.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout -s KILL 600 python bench.py --no-cpu-baseline > gpurun_out/bench_resnet50.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_resnet50.log | cut -c1-600
