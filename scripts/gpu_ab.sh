# A/B: build with each flag set ($@ = list of quoted flag sets), time the RN50 factor stage 3x each
cd /root/repo
for fl in "$@"; do
  KFAC_NVCC_EXTRA="$fl" python -c "import sys; sys.path.insert(0,'paper_1811_12019_b200'); import build; build.build(force=True)" > /dev/null 2>&1
  for r in 1 2 3; do echo "[$fl] $(timeout 120 python scripts/time_factor_all.py resnet50)"; done
done
python paper_1811_12019_b200/build.py > /dev/null
