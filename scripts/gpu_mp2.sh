cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
for a in "small 0" "small 1" "one_layer 0"; do
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29631 tests/mp_parity.py $a > gpurun_out/mp_$$.log 2>&1; echo "mp $a rc=$?"; grep mp_parity gpurun_out/mp_$$.log; grep -i "error" gpurun_out/mp_$$.log | head -3
done
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29632 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench2.log 2>&1; echo "bench2 rc=$?"
tail -c 600 gpurun_out/bench2.log
