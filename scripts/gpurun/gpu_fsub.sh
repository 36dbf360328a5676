cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 300 python scripts/factor_subset.py tensor
timeout -s KILL 300 python scripts/factor_subset.py all
timeout -s KILL 900 ncu --set full --clock-control none -k regex:factor_syrk -c 1 -o gpurun_out/prof_factor_tensor -f python scripts/factor_subset.py tensor 1 > gpurun_out/ncu_fsub.log 2>&1; echo "ncu rc=$?"
