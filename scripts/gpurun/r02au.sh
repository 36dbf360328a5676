# 1 GPU: C-tile L2 prefetch knob (bench N=1, inverse stage), 2 runs each
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for H in 1 0 1 0; do
  KFAC_NVCC_EXTRA="-DKFAC_OZ_C_PREFETCH=$H" python paper_1811_12019_b200/build.py --force > /dev/null 2>&1
  timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-stale --no-cpu-baseline --no-e2e > gpurun_out/bench_p$H.log 2>&1
  tail -1 gpurun_out/bench_p$H.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PREFETCH=$H', d['value'], d['stage_ms']['inverse'])"
done
