#!/bin/bash
# K4 decomposition (skip bits) + ncu of k_tiled at the default tiles
mkdir -p gpurun_out; rm -f gpurun_out/k4_decomp.txt
for s in 0 1 2 3 4 8 15; do
  SYMM_DEBUG_SKIP=$s timeout 300 python bench.py --config ${CFG:-st27_128} --steps 300 --warmup 10 --no-cpu-baseline --variant tiled_atomic 2>&1 | tail -1 | python -c "
import sys,json
l=json.loads(sys.stdin.read()); print('skip=$s', l['ms_per_step'], l['roofline']['frac'])" >> gpurun_out/k4_decomp.txt
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tiled -c 1 -o gpurun_out/k4_prof -f python bench.py --variant tiled_atomic --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_k4.log 2>&1
ncu -i gpurun_out/k4_prof.ncu-rep --page details > gpurun_out/k4_prof_details.txt 2>&1
ncu -i gpurun_out/k4_prof.ncu-rep --page source --csv > gpurun_out/k4_prof_source.csv 2>&1
ncu -i gpurun_out/k4_prof.ncu-rep --page raw --csv > gpurun_out/k4_prof_raw.csv 2>&1
