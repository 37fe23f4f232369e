#!/bin/bash
# K4 (tiled_atomic) tile-size sweep on st27_128: nnz cap : window cap
mkdir -p gpurun_out; rm -f gpurun_out/k4.txt
for cfg in ${CFGS:-1536:768 3000:1200 4500:1600 6000:2048}; do
  IFS=: read -r nz w wk <<< "$cfg"
  timeout 300 python bench.py --config ${CFG:-st27_128} --steps 300 --warmup 10 --no-cpu-baseline --variant tiled_atomic --tile-nnz $nz --tile-window $w --tile-work ${wk:-1792} 2>&1 | tail -1 | python -c "
import sys,json
t=sys.stdin.read()
try:
  l=json.loads(t); print('nnz=$nz W=$w work=$wk', l.get('ms_per_step'), l.get('roofline',{}).get('frac'), l['schedule']['tiles'], l['schedule']['spill_entries'], l['schedule']['plan'])
except Exception: print('nnz=$nz W=$w FAILED', t[-300:])" >> gpurun_out/k4.txt 2>&1
done
