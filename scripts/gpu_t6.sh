cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 120 python scripts/one_inverse.py 576 64 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 32 -c 40 --csv --log-file gpurun_out/inv576.csv python scripts/one_inverse.py 576 64 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
