# 1 GPU: bench lines of BASELINE configs 2 (RN18-CIFAR, batch 128) and 5 (stress) at HEAD
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
for C in resnet18_cifar stress; do
timeout -s KILL 600 python bench.py --config $C --no-cpu-baseline > gpurun_out/bench_$C.log 2>&1; echo "bench $C rc=$?"
tail -1 gpurun_out/bench_$C.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['stage_ms'], d['roofline']['frac'], d['clocks'])"
done
