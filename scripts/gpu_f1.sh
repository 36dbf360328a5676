cd /root/repo
python paper_1811_12019_b200/build.py > /dev/null
for m in 0 1 2 5; do KFAC_DBG_MODE=$m python scripts/time_factor_all.py resnet50; done
python scripts/prof_layers.py resnet50
