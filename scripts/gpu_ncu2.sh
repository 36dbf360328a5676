cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
KFAC_DBG_MODE=2 timeout -s KILL 120 python scripts/one_factor.py 44 A 3 > gpurun_out/one.log 2>&1 && \
KFAC_DBG_MODE=2 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:factor_syrk -s 2 -c 1 -o gpurun_out/prof_f44_dbg2 python scripts/one_factor.py 44 A 3 > gpurun_out/ncu_f.log 2>&1; echo "ncu1 rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:factor_syrk -s 2 -c 1 -o gpurun_out/prof_f44 python scripts/one_factor.py 44 A 3 > gpurun_out/ncu_f2.log 2>&1; echo "ncu2 rc=$?"
