cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
KFAC_DBG_MODE=1 timeout -s KILL 120 python scripts/one_factor.py 2 A 3 > gpurun_out/one.log 2>&1 && \
KFAC_DBG_MODE=1 timeout -s KILL 600 ncu --set full --clock-control none -k regex:factor_syrk -s 2 -c 1 -o gpurun_out/prof_f2_dbg1 python scripts/one_factor.py 2 A 3 > gpurun_out/ncu_f.log 2>&1; echo "ncu1 rc=$?"
