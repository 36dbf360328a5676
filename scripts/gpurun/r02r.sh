# 4 GPUs: bench N = 4 (auto / fp64 inverse) and N = 2
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
for A in "4 auto" "4 fp64" "2 auto"; do set -- $A
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 2957$1 bench.py --gpus $1 --inv-precision $2 --no-stale > gpurun_out/bench_n$1_$2.log 2>&1; echo "bench $1 $2 rc=$?"
tail -1 gpurun_out/bench_n$1_$2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['value'], d['stage_ms'], d['e2e']['value'])"
done
