#!/bin/bash
# FEM-like (fem_knn_4M) K4 sweep: schedule knobs and variants; ARGS entries are ';'-separated bench argument sets
mkdir -p gpurun_out; rm -f gpurun_out/fem.txt
IFS=';' read -ra SETS <<< "${ARGS:---variant tiled_atomic;--variant tiled}"
for args in "${SETS[@]}"; do
  timeout 400 python bench.py --config ${CFG:-fem_knn_4M} --steps 300 --warmup 10 --no-cpu-baseline $args 2>&1 | tail -1 | python -c "
import sys,json
t=sys.stdin.read()
try:
  l=json.loads(t); print('$args |', round(l['ms_per_step'],4), round(l['roofline']['frac'],3), 'tiles', l['schedule']['tiles'], 'spill', l['schedule'].get('spill_entries'), l['schedule'].get('plan'))
except Exception: print('$args FAILED', t[-300:])" >> gpurun_out/fem.txt 2>&1
done
cat gpurun_out/fem.txt
