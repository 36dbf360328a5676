cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout -s KILL 60 ./scripts/micro/tile_bench 2>&1 | head -2
timeout -s KILL 30 ./scripts/micro/pivot_test_dbg 128 0 | tail -16
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for n in "576 64" "2304 256" "4608 512"; do timeout -s KILL 120 python scripts/one_inverse.py $n 2>&1 | grep inverse; done
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print(d['value'], d['stage_ms'], d['factor_tflops'], d['roofline']['frac'], d['e2e']['value'])"
