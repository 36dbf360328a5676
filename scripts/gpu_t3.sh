cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for L in "13 G" "44 A" "2 A" "12 A" "47 A"; do
for m in 0 1 2; do KFAC_DBG_MODE=$m timeout -s KILL 60 python scripts/time_factor.py $L 2>&1 | tail -1; done
done
timeout -s KILL 300 python scripts/prof_layers.py resnet50 > gpurun_out/prof_layers.log 2>&1; tail -1 gpurun_out/prof_layers.log
