# round 2, first check: full-size step parity (RN50 x2 gamma, stress, RN18), all GPU tests, smoke, bench N=1 of configs 2, 3, 5
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; nproc > gpurun_out/nproc.txt
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 2400 python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/pytest_fullsize.log 2>&1; echo "fullsize rc=$?"; grep -E "worst|passed|failed|Error" gpurun_out/pytest_fullsize.log | tail -8
timeout -s KILL 1200 python -m pytest tests -q -m gpu --deselect tests/test_gpu_fullsize.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for c in resnet50 resnet18_cifar stress; do
timeout -s KILL 900 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?"; tail -1 gpurun_out/bench_$c.log | cut -c1-400
done
