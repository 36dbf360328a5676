# ONE ncu --set full capture of the persistent inverse inside an RN50 step
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 300 python scripts/step_once.py resnet50 1 > /dev/null 2>&1; echo "plain rc=$?"
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:inverse_kernel -c 1 \
  -o gpurun_out/prof_inv_r02ab -f python scripts/step_once.py resnet50 1 > gpurun_out/ncu_inv.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_inv.log
