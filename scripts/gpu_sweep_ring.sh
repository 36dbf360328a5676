# ring depth / chunk rows sweep of the inverse tile product (RN50 bench inverse stage + n=4608)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cfg in "8 4" "8 5" "12 3" "4 8" "16 2"; do
  set -- $cfg
  KFAC_NVCC_EXTRA="-DKFAC_INV_KC=$1 -DKFAC_INV_STAGES=$2" python -c "import sys; sys.path.insert(0,'paper_1811_12019_b200'); import build; build.build(force=True)" > /dev/null 2>&1 || { echo "build $cfg failed"; continue; }
  r=$(timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms']['inverse'])")
  i=$(timeout -s KILL 120 python scripts/one_inverse.py 4608 512 2>&1 | tail -1)
  echo "KC=$1 stages=$2: step/inverse $r | $i"
done
