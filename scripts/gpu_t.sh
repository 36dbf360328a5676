cd $GRAFT_REPO_ROOT
for L in "47 A" "12 A" "44 A" "2 A" "13 G"; do
for m in 0 2; do KFAC_DBG_MODE=$m timeout -s KILL 60 python scripts/time_factor.py $L 2>&1 | tail -1; done; done
