# 1 GPU: pivot phase cycles
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
KFAC_NVCC_EXTRA="-DPIVOT_DBG" python paper_1811_12019_b200/build.py --force > /dev/null 2>&1
timeout -s KILL 300 python scripts/pivot_phases.py > gpurun_out/pivot_phases.txt 2>&1; cat gpurun_out/pivot_phases.txt | tail -22
