# final check at HEAD (4 GPUs): every GPU test (incl. the P=4 legs), bench N=4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu4.log
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29574 bench.py --gpus 4 > gpurun_out/bench_n4.log 2>&1; echo "bench4 rc=$?"; tail -1 gpurun_out/bench_n4.log | cut -c1-200
