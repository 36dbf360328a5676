cd /root/repo
python paper_1811_12019_b200/build.py > /dev/null
for L in "44 A" "12 A" "2 A" "3 G" "47 A" "45 G"; do
for m in 0 1 2 4; do KFAC_DBG_MODE=$m python scripts/time_factor.py $L resnet50; done
done
