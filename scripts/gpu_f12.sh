cd /root/repo
python paper_1811_12019_b200/build.py > /dev/null
ncu --set full --import-source on -k regex:im2col -c 1 -o gpurun_out/prof_im2col -f python scripts/time_factor_all.py resnet50 > /dev/null 2>&1
ncu -i gpurun_out/prof_im2col.ncu-rep --page details --csv 2>/dev/null | grep -E "Duration|Throughput|Memory \[%\]|DRAM|L1/TEX Hit|L2 Hit|Warp Cycles Per Issued|Issue Slots|Eligible|Achieved Occupancy|Registers|Stall" | head -40
