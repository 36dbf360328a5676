# round-2 evidence (1 GPU): smoke, every GPU test (full-size parity included), bench (cpu baseline = full oracle step),
# reference arm, ncu launch list of the bench command, ONE ncu --set full capture of the hot kernels
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; nproc > gpurun_out/nproc.txt
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
S=$(date +%s); timeout -s KILL 1200 python bench.py > gpurun_out/bench_n1.log 2>&1; echo "bench rc=$? $(( $(date +%s) - S )) s"; tail -1 gpurun_out/bench_n1.log | cut -c1-400
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-300
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-stale > gpurun_out/ncu.log 2>&1; echo "ncu list rc=$?"
timeout -s KILL 1500 ncu --set full --clock-control none --import-source on -k "regex:factor_syrk|inverse_kernel|gemm_3xtf32" -c 4 \
  -o gpurun_out/prof_hot_rn50 -f python scripts/step_once.py resnet50 1 > gpurun_out/ncu_a.log 2>&1; echo "ncu full rc=$?"
