# bench lines N=1/2/4 (default flags)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 900 python bench.py > gpurun_out/bench_n1.log 2>&1; echo "bench1 rc=$?"
for N in 2 4; do
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N bench.py --gpus $N > gpurun_out/bench_n$N.log 2>&1; echo "bench$N rc=$?"
done
for N in 1 2 4; do tail -1 gpurun_out/bench_n$N.log | cut -c1-120; done
