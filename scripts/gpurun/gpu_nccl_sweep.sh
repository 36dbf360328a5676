# NCCL settings sweep for the RS / AG stages at N=4 (bench --no-e2e --no-cpu-baseline)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
for envs in "X=1" "NCCL_NVLS_ENABLE=0" "NCCL_MIN_NCHANNELS=32" "NCCL_ALGO=Ring" "NCCL_PROTO=Simple"; do
  env $envs timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29655 bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/nccl_sweep.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/nccl_sweep.log').read().strip().splitlines()[-1]); print('$envs', d['value'], d['stage_ms'])" 2>&1 | tail -1
done
NCCL_DEBUG=INFO timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29656 bench.py --gpus 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/nccl_debug.log 2>&1
grep -iE "NVLS|algo|channels" gpurun_out/nccl_debug.log | head -12
