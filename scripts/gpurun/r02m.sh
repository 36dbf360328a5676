# 4 GPUs: multi-GPU parity (NCCL paths, P = 2 / 4, RN50 and stress legs), bench N = 2 / 4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 2400 python -m pytest tests/test_multi_gpu.py -q -s > gpurun_out/pytest_mgpu4.log 2>&1; echo "pytest rc=$?"; grep -E "mp_parity|passed|failed" gpurun_out/pytest_mgpu4.log | tail -12
for N in 2 4; do
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N > gpurun_out/bench_n$N.log 2>&1; echo "bench$N rc=$?"
tail -1 gpurun_out/bench_n$N.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['value'], d['stage_ms'], d['e2e']['value'])"
done
