# NEXT-3 check: update GPU tests, bench line (stale + update keys), ncu --set full of the diff / update kernels
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 900 python -m pytest tests -x -q -m gpu -s -k "update" > gpurun_out/pytest_update.log 2>&1; echo "pytest update rc=$?"; tail -2 gpurun_out/pytest_update.log
timeout -s KILL 900 python bench.py --no-cpu-baseline > gpurun_out/bench_n1.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_n1.log | cut -c1-200
timeout -s KILL 600 python scripts/next_once.py > gpurun_out/next_once.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k "regex:diff_partial|update_step|update_scale" -c 3 \
  -o gpurun_out/prof_next -f python scripts/next_once.py > gpurun_out/ncu_next.log 2>&1; echo "ncu rc=$?"
