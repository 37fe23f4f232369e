#!/bin/bash
# NEXT-3: RACE vs MC vs ABMC schedules on the colored (K2) and tiled_atomic (K4) kernels, + DRAM bytes
mkdir -p gpurun_out; rm -f gpurun_out/mc.txt
for sch in "0" "1" "2:64" "2:256"; do
  IFS=: read -r sc bl <<< "$sch"
  for v in colored tiled_atomic; do
    timeout 600 python bench.py --config ${CFG:-st27_128} --steps 200 --warmup 5 --no-cpu-baseline --variant $v --sched scheme=$sc --sched abmc_block=${bl:-64} 2>/dev/null | tail -1 | python -c "
import sys,json
t=sys.stdin.read()
try:
  l=json.loads(t); print('scheme=$sc block=$bl $v', l['ms_per_step'], l['roofline']['frac'], 'phases', l['schedule']['phases'], 'colours/levels', l['schedule']['levels'], 'tiles', l['schedule']['tiles'])
except Exception: print('scheme=$sc $v FAILED', t[-300:])" >> gpurun_out/mc.txt
    timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_colored|k_tiled" -c 40 --csv --log-file gpurun_out/mc_ncu_${sc}_${bl}_${v}.csv python bench.py --config ${CFG:-st27_128} --steps 3 --warmup 2 --no-cpu-baseline --variant $v --sched scheme=$sc --sched abmc_block=${bl:-64} > /dev/null 2>&1
  done
done
