# 4 GPUs: bench N=4 and N=2 at HEAD (default flags), fast multi-GPU parity legs
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py --force > /dev/null
for N in 4 2; do
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2959$N bench.py --gpus $N > gpurun_out/bench_n$N.log 2>&1; echo "bench $N rc=$?"
tail -1 gpurun_out/bench_n$N.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['value'], d['stage_ms'], d['stage_ms_critical_rank'], d['e2e']['value'], d['clocks'])"
done
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29595 bench.py --gpus 4 --inv-precision fp64 --no-stale > gpurun_out/bench_n4_fp64.log 2>&1; echo "bench fp64 rc=$?"
tail -1 gpurun_out/bench_n4_fp64.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['value'], d['stage_ms'])"
timeout -s KILL 1500 python -m pytest tests/test_multi_gpu.py -q -s -k "small or one_layer" > gpurun_out/pytest_mgpu.log 2>&1; echo "pytest rc=$?"; grep -E "mp_parity.*policy|passed|failed" gpurun_out/pytest_mgpu.log | tail -12
