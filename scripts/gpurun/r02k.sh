# inverse tests + trace + bench
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -k "inverse" > gpurun_out/pytest_inv.log 2>&1; echo "inv rc=$?"; tail -2 gpurun_out/pytest_inv.log
bash scripts/gpurun/r02h.sh
