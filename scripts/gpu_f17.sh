cd /root/repo
KFAC_NVCC_EXTRA="-DKFAC_FACTOR_PROF" python -c "import sys; sys.path.insert(0,'paper_1811_12019_b200'); import build; build.build(force=True)" > /dev/null 2>&1
for m in 0 2; do echo "== dbg $m"; KFAC_DBG_MODE=$m python scripts/time_factor_all.py resnet50 2>&1 | grep -E "fprof|factors" | head -7; done
for pat in "l3b[1-5]c2" "l1b.c2" "c[13]$|ds"; do echo "== $pat"; python scripts/time_factor_sub.py resnet50 "$pat" 2>&1 | grep -E "fprof|factors" | grep -E "warp 8|factors" | head -3; done
