cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 60 ./scripts/micro/tile_bench 2>&1 | head -3
timeout -s KILL 600 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b1.log 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 246 -c 90 --csv --log-file gpurun_out/launches_step.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
