cd /root/repo
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/mma_bench scripts/micro/mma_bench.cu && /tmp/mma_bench
python paper_1811_12019_b200/build.py > /dev/null
for m in 4 2; do KFAC_DBG_MODE=$m python scripts/time_factor_all.py resnet50; done
KFAC_DEBUG=1 python scripts/time_factor_all.py resnet50 2>&1 | grep -E "launch|prob" | head -120
