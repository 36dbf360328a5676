cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 120 python scripts/one_inverse.py 4608 512 > /dev/null 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:update_kernel -s 80 -c 1 -o gpurun_out/prof_update2 python scripts/one_inverse.py 4608 512 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
