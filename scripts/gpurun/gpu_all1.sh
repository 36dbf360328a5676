# 1 GPU: every GPU test, the default bench line, ncu of the BN kernels (bench-shaped)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 1200 python -m pytest tests -x -q -m gpu -s > gpurun_out/pytest_all1.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_all1.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_n1.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_n1.log | cut -c1-200
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "regex:bn_|diff_|update_" --csv --log-file gpurun_out/next_kernels.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_nk.log 2>&1; echo "ncu rc=$?"
