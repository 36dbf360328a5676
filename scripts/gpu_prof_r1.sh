cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b1.log 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 246 -c 90 --csv --log-file gpurun_out/launches_step.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:factor_syrk -s 3 -c 1 -o gpurun_out/prof_factor_rn50 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:update_kernel -s 110 -c 1 -o gpurun_out/prof_update_rn50 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu3.log 2>&1; echo "ncu3 rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32 -s 6 -c 1 -o gpurun_out/prof_gemm_rn50 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu4.log 2>&1; echo "ncu4 rc=$?"
