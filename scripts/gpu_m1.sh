cd /root/repo
for mm in 0 1 2; do echo "== mbar mode $mm"; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DKFAC_MBAR_MODE=$mm -o /tmp/mlb scripts/micro/mma_loop_bench.cu && timeout 60 /tmp/mlb; done
