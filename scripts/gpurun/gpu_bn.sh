# NEXT-2 check: BN GPU tests, bench line (bn_fisher key), ncu --set full of the BN kernels
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 900 python -m pytest tests -x -q -m gpu -s -k "bn" > gpurun_out/pytest_bn.log 2>&1; echo "pytest bn rc=$?"; tail -2 gpurun_out/pytest_bn.log
timeout -s KILL 900 python bench.py --no-cpu-baseline > gpurun_out/bench_n1.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_n1.log | cut -c1-200
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k "regex:bn_grads|bn_precond" -c 3 \
  -o gpurun_out/prof_bn -f python -m pytest tests/test_gpu_bn.py -x -q -k resnet50 > gpurun_out/ncu_bn.log 2>&1; echo "ncu rc=$?"
