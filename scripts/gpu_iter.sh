cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -q -s -p no:cacheprovider -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|err|Error" gpurun_out/pytest_gpu.log | tail -40
for L in "47 A" "12 A" "44 A" "2 A" "0 A"; do
for m in 0 2; do KFAC_DBG_MODE=$m timeout -s KILL 60 python scripts/time_factor.py $L 2>&1 | tail -1; done; done
timeout -s KILL 300 python scripts/prof_layers.py resnet50 > gpurun_out/prof_layers.log 2>&1; tail -1 gpurun_out/prof_layers.log
