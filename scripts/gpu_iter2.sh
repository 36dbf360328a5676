# build, GPU parity tests, then a short bench (RN50 1 GPU)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 900 python -m pytest tests -q -m gpu -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAIL|Error|residual|cond=" gpurun_out/pytest_gpu.log | tail -30
timeout -s KILL 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log | cut -c1-900
timeout -s KILL 120 python scripts/one_inverse.py 4608 512 2>&1 | tail -1
