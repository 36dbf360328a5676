cd /root/repo
python paper_1811_12019_b200/build.py > /dev/null
timeout 300 python scripts/check_factors.py | tail -1
timeout 120 python scripts/time_factor_all.py resnet50
bash scripts/gpu_f11.sh 2>&1 | tail -4
KFAC_NVCC_EXTRA="-DKFAC_FACTOR_PROF" python -c "import sys; sys.path.insert(0,'paper_1811_12019_b200'); import build; build.build(force=True)" > /dev/null 2>&1
for m in 0 2; do echo "== dbg $m"; KFAC_DBG_MODE=$m python scripts/time_factor_all.py resnet50 2>&1 | grep -E "fprof|factors" | head -7; done
