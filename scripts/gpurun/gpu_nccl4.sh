# 4 GPUs: isolated NCCL RS (sum vs avg) / AG at the RN50 plan's chunk sizes, NVLS check, bench N=4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
for N in 2 4; do
NCCL_DEBUG=INFO timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=2966$N scripts/nccl_rs_bench.py > gpurun_out/nccl_rs_$N.log 2>&1; echo "nccl$N rc=$?"
grep -E "^(rs|ag) " gpurun_out/nccl_rs_$N.log; grep -ciE "NVLS" gpurun_out/nccl_rs_$N.log
done
grep -iE "NVLS" gpurun_out/nccl_rs_4.log | head -5
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29554 bench.py --gpus 4 > gpurun_out/bench_n4.log 2>&1; echo "bench4 rc=$?"
tail -1 gpurun_out/bench_n4.log | cut -c1-200
