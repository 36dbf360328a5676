cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 120 python scripts/one_factor.py 47 A 3 > gpurun_out/one.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:factor_syrk -s 2 -c 1 -o gpurun_out/prof_factor_l4b1c1 python scripts/one_factor.py 47 A 3 > gpurun_out/ncu_f.log 2>&1; echo "ncu1 rc=$?"
timeout -s KILL 120 python scripts/one_factor.py 12 A 3 > gpurun_out/one2.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:factor_syrk -s 2 -c 1 -o gpurun_out/prof_factor_l2b0c2 python scripts/one_factor.py 12 A 3 > gpurun_out/ncu_f2.log 2>&1; echo "ncu2 rc=$?"
timeout -s KILL 120 python scripts/one_inverse.py 2304 > gpurun_out/inv.log 2>&1; cat gpurun_out/inv.log
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"update_kernel|pivot_kernel" -s 60 -c 2 -o gpurun_out/prof_inverse python scripts/one_inverse.py 2304 > gpurun_out/ncu_i.log 2>&1; echo "ncu3 rc=$?"
ls -la gpurun_out
