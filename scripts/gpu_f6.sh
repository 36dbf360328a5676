cd /root/repo
python paper_1811_12019_b200/build.py > /dev/null
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -15
for m in 0 4 2 1; do KFAC_DBG_MODE=$m timeout 120 python scripts/time_factor_all.py resnet50; done
KFAC_DEBUG=1 timeout 120 python scripts/time_factor_all.py resnet50 2>&1 | grep -E "launch" | head
