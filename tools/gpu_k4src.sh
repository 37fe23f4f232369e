#!/bin/bash
# ncu source-level capture of k_tiled (st27 by default) under an optional env setting (ENV='K=V')
mkdir -p gpurun_out; C=${CFG:-st27_128}; T=${TAG:-x}
( [ -n "$ENV" ] && export $ENV; timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tiled -c 1 -o gpurun_out/k4src_${C}_$T -f python bench.py --config $C --variant tiled_atomic --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/k4src_${C}_$T.log 2>&1 )
ncu -i gpurun_out/k4src_${C}_$T.ncu-rep --page source --csv > gpurun_out/k4src_${C}_${T}_source.csv 2>&1
