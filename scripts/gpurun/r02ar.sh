# 1 GPU: dependency-poll sleep sweep (bench N=1, inverse stage)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for NS in 200 50 20; do
  KFAC_NVCC_EXTRA="-DKFAC_WAIT_NS=$NS" python paper_1811_12019_b200/build.py --force > /dev/null 2>&1
  timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-stale --no-cpu-baseline --no-e2e > gpurun_out/bench_ns$NS.log 2>&1
  tail -1 gpurun_out/bench_ns$NS.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NS=$NS', d['value'], d['stage_ms']['inverse'])"
done
