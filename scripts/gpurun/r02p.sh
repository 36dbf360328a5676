# bisect the inverse variants: TMEM sets 2/3, packed first touch on/off (bench inverse stage)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for V in "-DKFAC_OZ_SETS=3 -DKFAC_OZ_FIRST_TOUCH=1" "-DKFAC_OZ_SETS=2 -DKFAC_OZ_FIRST_TOUCH=1" "-DKFAC_OZ_SETS=3 -DKFAC_OZ_FIRST_TOUCH=0" "-DKFAC_OZ_SETS=2 -DKFAC_OZ_FIRST_TOUCH=0"; do
KFAC_NVCC_EXTRA="$V" python -c "import sys; sys.path.insert(0,'paper_1811_12019_b200'); import build; build.build(force=True)" > /dev/null 2>&1
timeout -s KILL 300 python bench.py --no-cpu-baseline --no-e2e --no-stale --steps 10 > gpurun_out/b.log 2>&1
echo "$V: $(tail -1 gpurun_out/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stage_ms'])")"
done
