# 1 GPU: digit-cut lane mapping sweep (trace timings), parity of each variant
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for L in 2 4 1; do
  KFAC_NVCC_EXTRA="-DKFAC_OZ_SLICE_LANES=$L" python paper_1811_12019_b200/build.py --force > /dev/null 2>&1
  timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k "inverse" > gpurun_out/pytest_inv_$L.log 2>&1; echo "L=$L inverse tests rc=$?"
  timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-stale > gpurun_out/bench_$L.log 2>&1
  tail -1 gpurun_out/bench_$L.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('L=$L', d['value'], d['stage_ms']['inverse'])"
  KFAC_NVCC_EXTRA="-DINV_TRACE -DKFAC_OZ_SLICE_LANES=$L" python paper_1811_12019_b200/build.py --force > /dev/null 2>&1
  timeout -s KILL 600 python scripts/trace_step.py gpurun_out/trace_$L.txt > /dev/null 2>&1
  python scripts/trace_analyze.py gpurun_out/trace_$L.txt 2>&1 | grep -E "kind 0 detail|kind 5 epi|total"
done
