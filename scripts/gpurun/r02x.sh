# 4 GPUs: bench N = 4 and N = 2 with NUMA-bound host buffers; fast multi-GPU parity legs
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
for N in 4 2; do
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2958$N bench.py --gpus $N > gpurun_out/bench_n$N.log 2>&1; echo "bench $N rc=$?"
tail -1 gpurun_out/bench_n$N.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['value'], d['stage_ms'], d['e2e']['value'], d['config'].get('host_numa_node'), d.get('stale',{}).get('amortized_ms'))"
done
timeout -s KILL 1200 python -m pytest tests/test_multi_gpu.py -q -s -k "small or one_layer or (resnet50 and 2 and 0)" > gpurun_out/pytest_mgpu4.log 2>&1; echo "pytest rc=$?"; grep -E "mp_parity.*policy|passed|failed" gpurun_out/pytest_mgpu4.log | tail -8
