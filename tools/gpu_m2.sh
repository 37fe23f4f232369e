#!/bin/bash
mkdir -p gpurun_out
timeout 120 ./tools/micro2 > gpurun_out/micro2.txt 2>&1
SYMM_CS_WINDOW=2048 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_cs -c 1 -o gpurun_out/cs_w2048 -f python bench.py --variant colored_smem --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_cs.log 2>&1
ncu -i gpurun_out/cs_w2048.ncu-rep --page details > gpurun_out/cs_w2048_details.txt 2>&1
