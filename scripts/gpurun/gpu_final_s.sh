# final check at HEAD (2 GPUs): every GPU test, smoke(), bench N=1 and N=2, launch list of one step
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout -s KILL 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu2.log
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 900 python bench.py > gpurun_out/bench_n1.log 2>&1; echo "bench1 rc=$?"; tail -1 gpurun_out/bench_n1.log | cut -c1-300
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29572 bench.py --gpus 2 > gpurun_out/bench_n2.log 2>&1; echo "bench2 rc=$?"; tail -1 gpurun_out/bench_n2.log | cut -c1-200
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:inverse|finalize|pivot" -c 60 --csv --log-file gpurun_out/launches_inv.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
