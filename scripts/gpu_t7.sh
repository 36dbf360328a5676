cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for n in 33 128; do timeout -s KILL 30 ./scripts/micro/pivot_test $n | tail -1; done
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for n in "576 64" "2304 256" "4608 512"; do timeout -s KILL 120 python scripts/one_inverse.py $n 2>&1 | grep inverse; done
timeout -s KILL 120 python scripts/one_inverse.py 576 64 > /dev/null 2>&1 && timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 32 -c 40 --csv --log-file gpurun_out/inv576.csv python scripts/one_inverse.py 576 64 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
