cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 120 python scripts/one_inverse.py 4608 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active --clock-control none -s 220 -c 110 --csv --log-file gpurun_out/inv_launches.csv python scripts/one_inverse.py 4608 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
