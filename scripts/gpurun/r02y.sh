# 2 GPUs: fp16 wire parity (1-GPU tests + P=2 mp legs) and bench N=2 fp32 vs fp16 wire
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 900 python -m pytest tests/test_gpu_wire.py -q -s -x > gpurun_out/pytest_wire.log 2>&1; echo "wire tests rc=$?"; tail -5 gpurun_out/pytest_wire.log; grep "end-to-end" gpurun_out/pytest_wire.log
for leg in "small 1 1 1" "one_layer 0 1 1" "small 1 0 1"; do
  set -- $leg
  timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 tests/mp_parity.py $1 $2 $3 $4 > gpurun_out/mp_$1_$3_$4.log 2>&1; echo "mp $leg rc=$?"; grep "mp_parity" gpurun_out/mp_$1_$3_$4.log
done
for W in fp32 fp16; do
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29582 bench.py --gpus 2 --wire $W > gpurun_out/bench_n2_$W.log 2>&1; echo "bench $W rc=$?"
tail -1 gpurun_out/bench_n2_$W.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['value'], d['stage_ms'], d['e2e']['value'])"
done
