# 1 GPU: inverse + precondition + stale tests, full-size parity, trace, bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stale.py -x -q > gpurun_out/pytest_inv.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/pytest_inv.log
timeout -s KILL 1800 python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/pytest_fullsize.log 2>&1; echo "fullsize rc=$?"; grep -E "worst|passed|failed|Error" gpurun_out/pytest_fullsize.log | tail -6
bash scripts/gpurun/r02h.sh
