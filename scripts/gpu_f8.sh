cd /root/repo
for L in 1 2 4 8; do
KFAC_NVCC_EXTRA="-DKFAC_ISSUE_LANES=$L" python -c "import sys; sys.path.insert(0,'paper_1811_12019_b200'); import build; build.build(force=True)" > /dev/null 2>&1
echo "== lanes $L"; for m in 0 1; do KFAC_DBG_MODE=$m python scripts/time_factor_all.py resnet50 2>&1 | grep factors; done
done
