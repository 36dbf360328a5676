cd $GRAFT_REPO_ROOT
for L in "13 G" "44 A" "2 A"; do
for m in 0 2 3 4 5; do KFAC_DBG_MODE=$m timeout -s KILL 60 python scripts/time_factor.py $L 2>&1 | tail -1; done
KFAC_NO_FIXUP=1 timeout -s KILL 60 python scripts/time_factor.py $L 2>&1 | tail -1 | sed 's/^/nofixup /'
done
