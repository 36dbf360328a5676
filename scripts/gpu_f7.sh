cd /root/repo
KFAC_NVCC_EXTRA="-DKFAC_FACTOR_PROF" python -c "import sys; sys.path.insert(0,'paper_1811_12019_b200'); import build; build.build(force=True)" > /dev/null 2>&1
for m in 0 2 4; do echo "== dbg $m"; KFAC_DBG_MODE=$m python scripts/time_factor_all.py resnet50 2>&1 | grep -E "fprof|factors" | head -12; done
