# round evidence (1 GPU): pytest -m gpu, bench JSON line (+ e2e, cpu_baseline), reference arm,
# ncu launch list of the bench command, ONE ncu --set full capture of the hot kernels
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_n1.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_n1.log | cut -c1-300
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-300
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-stale > gpurun_out/ncu.log 2>&1; echo "ncu list rc=$?"
timeout -s KILL 600 python scripts/step_once.py resnet50 1 > /dev/null 2>&1 && \
timeout -s KILL 1500 ncu --set full --clock-control none --import-source on -k "regex:factor_syrk|inverse_kernel|gemm_3xtf32" -c 4 \
  -o gpurun_out/prof_hot_rn50 -f python scripts/step_once.py resnet50 1 > gpurun_out/ncu_a.log 2>&1; echo "ncu full rc=$?"
