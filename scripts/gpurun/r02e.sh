# timeline of the int8-sliced inverse: RN50 step + a lone 4608 (INV_TRACE build)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
KFAC_NVCC_EXTRA=-DINV_TRACE python -c "import sys; sys.path.insert(0,'paper_1811_12019_b200'); import build; build.build(force=True)" > /dev/null 2>&1
timeout -s KILL 300 python scripts/trace_step.py gpurun_out/trace_step.txt; echo "trace rc=$?"
python scripts/trace_analyze.py gpurun_out/trace_step.txt | grep -v "^ *[0-9]" | tail -12
timeout -s KILL 300 python scripts/trace_one.py 4608 gpurun_out/trace_one.txt; echo "trace1 rc=$?"
python scripts/trace_analyze.py gpurun_out/trace_one.txt | tail -12
python paper_1811_12019_b200/build.py --force > /dev/null
timeout -s KILL 300 python scripts/one_inverse.py 4608 64
