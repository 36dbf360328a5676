# full-size step parity only
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 2400 python -m pytest tests/test_gpu_fullsize.py -q -s > gpurun_out/pytest_fullsize.log 2>&1; echo "fullsize rc=$?"; grep -E "worst|passed|failed|Error" gpurun_out/pytest_fullsize.log | tail -12
