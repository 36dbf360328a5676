# 4-GPU: NCCL parity (torchrun) + bench lines at N=2 and N=4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
for a in "small 1" "one_layer 0"; do
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29631 tests/mp_parity.py $a > gpurun_out/mp4.log 2>&1; echo "mp4 $a rc=$?"; grep mp_parity gpurun_out/mp4.log
done
timeout -s KILL 600 python -m pytest tests -q -m gpu -k multi > gpurun_out/pytest_multi.log 2>&1; echo "pytest multi rc=$?"; tail -1 gpurun_out/pytest_multi.log
for N in 2 4; do
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=2964$N bench.py --gpus $N > gpurun_out/bench_n$N.log 2>&1; echo "bench N=$N rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_n$N.log').read().strip().splitlines()[-1]); print(d['n_gpus'], d['value'], d['stage_ms'], d['e2e']['value'], d['clocks'])"
done
