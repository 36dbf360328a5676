cd /root/repo
for cfgw in "4 1" "2 1" "1 1" "4 2"; do set -- $cfgw
KFAC_NVCC_EXTRA="-DKFAC_PROD_WARPS=$1 -DKFAC_ISSUE_LANES=$2" python -c "import sys; sys.path.insert(0,'paper_1811_12019_b200'); import build; build.build(force=True)" > /dev/null 2>&1
echo "== warps $1 lanes $2"
for pat in "l1b.c2" "l2b.c2" "l3b.c2" "l4b.c2" "c[13]$|ds"; do for m in 0 1 2; do KFAC_DBG_MODE=$m python scripts/time_factor_sub.py resnet50 "$pat" 2>&1 | grep factors; done; done
done
