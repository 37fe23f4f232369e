#!/bin/bash
# K4 decomposition (skip bits; needs a build with make EXTRA_NVFLAGS=-DK4_DEBUG_SKIP) + ncu of k_tiled; CFG picks the config, NODECOMP=1 skips the sweep
mkdir -p gpurun_out; C=${CFG:-st27_128}; rm -f gpurun_out/k4_decomp_$C.txt
if [ -z "$NODECOMP" ]; then
for s in 0 1 2 3 4 8 15; do
  SYMM_DEBUG_SKIP=$s timeout 300 python bench.py --config $C --steps 300 --warmup 10 --no-cpu-baseline --variant tiled_atomic 2>&1 | tail -1 | python -c "
import sys,json
l=json.loads(sys.stdin.read()); print('skip=$s', l['ms_per_step'], l['roofline']['frac'])" >> gpurun_out/k4_decomp_$C.txt
done
fi
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tiled -c 1 -o gpurun_out/k4_prof_$C -f python bench.py --config $C --variant tiled_atomic --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_k4_$C.log 2>&1
ncu -i gpurun_out/k4_prof_$C.ncu-rep --page details > gpurun_out/k4_prof_${C}_details.txt 2>&1
ncu -i gpurun_out/k4_prof_$C.ncu-rep --page source --csv > gpurun_out/k4_prof_${C}_source.csv 2>&1
ncu -i gpurun_out/k4_prof_$C.ncu-rep --page raw --csv > gpurun_out/k4_prof_${C}_raw.csv 2>&1
