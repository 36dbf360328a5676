# per-task timeline of the persistent inverse inside one RN50 step (INV_TRACE build), + DMMA shapes
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
KFAC_NVCC_EXTRA=-DINV_TRACE python -c "import sys; sys.path.insert(0,'paper_1811_12019_b200'); import build; build.build(force=True)" > /dev/null 2>&1
timeout -s KILL 300 python scripts/trace_step.py gpurun_out/trace_step.txt; echo "trace rc=$?"
python scripts/trace_analyze.py gpurun_out/trace_step.txt | tail -8
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/dmma2 scripts/micro/dmma_bench2.cu && timeout 60 /tmp/dmma2
