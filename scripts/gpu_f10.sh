cd /root/repo
python paper_1811_12019_b200/build.py > /dev/null
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for m in 0 1 2; do KFAC_DBG_MODE=$m timeout 120 python scripts/time_factor_all.py resnet50; done
for pat in "l1b.c2" "l2b.c2" "l3b.c2" "l4b.c2" "c[13]$|ds"; do for m in 0 1; do KFAC_DBG_MODE=$m python scripts/time_factor_sub.py resnet50 "$pat" 2>&1 | grep factors; done; done
