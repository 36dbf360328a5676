# memcheck of the inverse on a small case
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python paper_1811_12019_b200/build.py > /dev/null
timeout -s KILL 300 python scripts/one_inverse.py 1153 64; echo "plain rc=$?"
timeout -s KILL 900 compute-sanitizer --tool memcheck --show-backtrace device --print-limit 20 python scripts/one_inverse.py 1153 64 > gpurun_out/memcheck_inv.log 2>&1; echo "memcheck rc=$?"
grep -v "^=========     " gpurun_out/memcheck_inv.log | head -40
