# 4 GPUs: bench N=4 (fp32 / fp16 wire) with the critical rank's stage split; fp16-wire parity legs at P=4
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
for W in fp32 fp16; do
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29584 bench.py --gpus 4 --wire $W > gpurun_out/bench_n4_$W.log 2>&1; echo "bench $W rc=$?"
tail -1 gpurun_out/bench_n4_$W.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['value'], d['stage_ms'], d['stage_ms_critical_rank'], d['e2e']['value'], d['clocks'])"
done
for leg in "small 1 0 1" "resnet50 1 1 1"; do
  set -- $leg
  timeout -s KILL 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29642 tests/mp_parity.py $1 $2 $3 $4 > gpurun_out/mp4_$1_$3_$4.log 2>&1; echo "mp $leg rc=$?"; grep "mp_parity" gpurun_out/mp4_$1_$3_$4.log
done
