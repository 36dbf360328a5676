cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
KFAC_NVCC_EXTRA=-DKFAC_FACTOR_PROF python -c "import sys; sys.path.insert(0,'paper_1811_12019_b200'); import build; build.build(force=True)" > /dev/null 2>&1
timeout -s KILL 300 python scripts/factor_subset.py tensor 1 2>&1 | tail -12
timeout -s KILL 300 python scripts/factor_subset.py all 1 2>&1 | tail -12
