#!/bin/bash
# A/B of environment settings (';'-separated ENVS, each 'K=V K2=V2' or 'none') on CFGS, tiled_atomic
mkdir -p gpurun_out; rm -f gpurun_out/envab.txt
IFS=';' read -ra SETS <<< "${ENVS:-none}"
for e in "${SETS[@]}"; do
  for c in ${CFGS:-st27_128 fem_knn_4M spin_22 lap3d_256}; do
    ( [ "$e" != none ] && export $e; timeout 400 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline --variant ${VARIANT:-tiled_atomic} 2>&1 | tail -1 | python -c "
import sys,json
t=sys.stdin.read()
try:
  l=json.loads(t); print('$e $c', round(l['ms_per_step'],4), round(l['roofline']['frac'],3), 'tiles', l['schedule']['tiles'], 'stages', l['schedule']['plan'].get('tiled_stages'), 'bcap', l['schedule']['plan'].get('block_cap'))
except Exception: print('$e $c FAILED', t[-300:])" ) >> gpurun_out/envab.txt 2>&1
  done
done
cat gpurun_out/envab.txt
