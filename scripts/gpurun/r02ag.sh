# 1 GPU: inverse trace summary (chain breakdown)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
KFAC_NVCC_EXTRA=-DINV_TRACE python paper_1811_12019_b200/build.py --force > /dev/null 2>&1
timeout -s KILL 600 python scripts/trace_step.py gpurun_out/trace.txt > gpurun_out/trace_run.log 2>&1; echo "trace rc=$?"
python scripts/trace_analyze.py gpurun_out/trace.txt > gpurun_out/trace_summary.txt 2>&1; grep -E "kind|total" gpurun_out/trace_summary.txt
