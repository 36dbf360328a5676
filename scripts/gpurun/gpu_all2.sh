# 2 GPUs: every GPU test (incl. the P=2 mp_parity legs: stale step, BN exchange), 1-GPU bench line, BN / NEXT kernel times
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 1200 python -m pytest tests -x -q -m gpu -s > gpurun_out/pytest_all2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_all2.log
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 900 python bench.py > gpurun_out/bench_n1.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_n1.log | cut -c1-200
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "regex:bn_|diff_|update_" --csv --log-file gpurun_out/next_kernels.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_nk.log 2>&1; echo "ncu rc=$?"
