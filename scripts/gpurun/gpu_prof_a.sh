# round profile, part A: the 1-GPU bench line, then ONE ncu --set full capture of the three
# hot kernels of one step (factor_syrk_kernel, inverse_kernel, gemm_3xtf32_kernel x2)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 900 python bench.py > gpurun_out/bench_n1.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_n1.log | cut -c1-300
timeout -s KILL 600 python scripts/step_once.py resnet50 1 > /dev/null 2>&1 && \
timeout -s KILL 1500 ncu --set full --clock-control none --import-source on -k "regex:factor_syrk|inverse_kernel|gemm_3xtf32" -c 4 \
  -o gpurun_out/prof_hot_rn50 -f python scripts/step_once.py resnet50 1 > gpurun_out/ncu_a.log 2>&1; echo "ncu rc=$?"
