#!/bin/bash
# ncu evidence of HEAD for the headline config: launch list of the default bench command and one
# ncu --set full capture of k_tiled on lap3d_512
mkdir -p gpurun_out/h2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/h2/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/h2/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tiled -c 1 -o gpurun_out/h2/k_tiled_lap3d_512 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/h2/ncu_full.log 2>&1
ncu -i gpurun_out/h2/k_tiled_lap3d_512.ncu-rep --page raw --csv > gpurun_out/h2/k_tiled_lap3d_512_raw.csv 2>&1
ncu -i gpurun_out/h2/k_tiled_lap3d_512.ncu-rep --page details > gpurun_out/h2/k_tiled_lap3d_512_details.txt 2>&1
grep -E "Duration|DRAM Throughput" gpurun_out/h2/k_tiled_lap3d_512_details.txt
