cd $GRAFT_REPO_ROOT
for n in "33 16" "64 16" "65 16" "96 16" "120 16"; do
  KFAC_INV_NOFUSE=1 timeout -s KILL 60 python scripts/one_inverse.py $n 2>&1 | grep -E "inverse|Error" | tail -1 | sed "s/^/nofuse $n: /"
done
