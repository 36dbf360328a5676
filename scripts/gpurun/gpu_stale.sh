# NEXT-1 check (2 GPUs): all GPU tests (incl. the stale-step mp_parity legs at P=2), then the 1-GPU bench line
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 900 python -m pytest tests -x -q -m gpu -s -k "stale or mp_parity" > gpurun_out/pytest_stale.log 2>&1; echo "pytest stale rc=$?"; tail -2 gpurun_out/pytest_stale.log
timeout -s KILL 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 900 python bench.py --no-cpu-baseline > gpurun_out/bench_n1.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_n1.log | cut -c1-300
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --no-e2e > gpurun_out/bench_n2.log 2>&1; echo "bench2 rc=$?"
