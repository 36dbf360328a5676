cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 300 python scripts/prof_layers.py resnet50 > gpurun_out/prof_layers.log 2>&1; echo "prof rc=$?"
cat gpurun_out/prof_layers.log | tail -60
KFAC_DEBUG=1 timeout -s KILL 300 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_dbg.log 2>&1; echo "bench rc=$?"
grep "factor launch" gpurun_out/bench_dbg.log | head -2
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 700 -c 260 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu.log
