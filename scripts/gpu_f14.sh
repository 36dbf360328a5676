cd /root/repo
KFAC_NVCC_EXTRA="-DKFAC_FACTOR_PROF" python -c "import sys; sys.path.insert(0,'paper_1811_12019_b200'); import build; build.build(force=True)" > /dev/null 2>&1
for m in 2 0; do echo "== dbg $m"; KFAC_DBG_MODE=$m python scripts/time_factor_sub.py resnet50 "l3b[1-5]c2" 2>&1 | grep -E "fprof|factors" | head -7; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/mma_bench scripts/micro/mma_bench.cu && /tmp/mma_bench
