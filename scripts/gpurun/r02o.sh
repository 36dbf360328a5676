# 2 GPUs: 1-GPU inverse/precondition/stale parity + full-size parity on GPU 0, small P=2 NCCL parity (both RS modes),
# bench N=1 (no cpu baseline) and N=2 (both RS modes)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
export CUDA_VISIBLE_DEVICES_ALL=$CUDA_VISIBLE_DEVICES
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stale.py -x -q > gpurun_out/pytest_inv.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/pytest_inv.log
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/pytest_fullsize.log 2>&1; echo "fullsize rc=$?"; grep -E "worst|passed|failed|Error" gpurun_out/pytest_fullsize.log | tail -6
timeout -s KILL 900 python -m pytest tests/test_multi_gpu.py -q -s -k "small and 2" > gpurun_out/pytest_mgpu2.log 2>&1; echo "mgpu rc=$?"; grep -E "mp_parity.*policy|passed|failed" gpurun_out/pytest_mgpu2.log | tail -6
CUDA_VISIBLE_DEVICES=0 timeout -s KILL 600 python bench.py --no-cpu-baseline > gpurun_out/bench_n1.log 2>&1; echo "bench1 rc=$?"
for M in padded per_owner; do
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 2 --rs-mode $M > gpurun_out/bench_n2_$M.log 2>&1; echo "bench2 $M rc=$?"
done
for f in bench_n1 bench_n2_padded bench_n2_per_owner; do tail -1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['value'], d['stage_ms'], d['e2e']['value'])"; done
