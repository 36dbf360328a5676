cd /root/repo
python paper_1811_12019_b200/build.py > /dev/null
timeout 300 python scripts/check_factors.py | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
KFAC_FORCE_GATHER=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "factor and not fullsize" 2>&1 | tail -2
for m in 0 2; do KFAC_DBG_MODE=$m timeout 120 python scripts/time_factor_all.py resnet50; done
