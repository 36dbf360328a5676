cd /root/repo
for mm in 0 1 2; do
  KFAC_NVCC_EXTRA="-DKFAC_MBAR_MODE=$mm" python -c "import sys; sys.path.insert(0,'paper_1811_12019_b200'); import build; build.build(force=True)" > /dev/null
  echo "== mbar mode $mm"
  for m in 0 4 2; do KFAC_DBG_MODE=$m python scripts/time_factor_all.py resnet50; done
done
