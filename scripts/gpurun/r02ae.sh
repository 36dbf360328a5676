# 4 GPUs: fp16-wire parity (1-GPU tests, P=2/4 legs), bench N=4 fp32 / fp16
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 900 python -m pytest tests/test_gpu_wire.py -q -s -x > gpurun_out/pytest_wire.log 2>&1; echo "wire tests rc=$?"; tail -2 gpurun_out/pytest_wire.log; grep "end-to-end" gpurun_out/pytest_wire.log
for leg in "2 small 1 1 1" "4 small 1 0 1" "4 resnet50 1 1 1"; do
  set -- $leg
  timeout -s KILL 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 29643 tests/mp_parity.py $2 $3 $4 $5 > gpurun_out/mp$1_$2_$4_$5.log 2>&1; echo "mp $leg rc=$?"; grep "mp_parity" gpurun_out/mp$1_$2_$4_$5.log
done
for W in fp32 fp16; do
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29585 bench.py --gpus 4 --wire $W > gpurun_out/bench_n4_$W.log 2>&1; echo "bench $W rc=$?"
tail -1 gpurun_out/bench_n4_$W.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['value'], d['stage_ms'], d['stage_ms_critical_rank'], d['e2e']['value'], d['clocks'])"
done
