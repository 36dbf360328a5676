# 4 GPUs: final bench N=4 / N=2 at HEAD (default flags), stress at N=4, fast parity legs
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
for N in 4 2; do
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N bench.py --gpus $N > gpurun_out/bench_n$N.log 2>&1; echo "bench $N rc=$?"
tail -1 gpurun_out/bench_n$N.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['value'], d['stage_ms'], d['stage_ms_critical_rank'], d['e2e']['value'], d['clocks'])"
done
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29617 bench.py --gpus 4 --config stress --no-stale > gpurun_out/bench_stress_n4.log 2>&1; echo "stress rc=$?"
tail -1 gpurun_out/bench_stress_n4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['value'], d['stage_ms_critical_rank'])"
timeout -s KILL 900 python -m pytest tests/test_multi_gpu.py -q -s -k "small or one_layer" > gpurun_out/pytest_mgpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_mgpu.log
