#!/bin/bash
# Evidence of HEAD (tests, smoke, bench lines, launch list, ncu) + one schedule experiment:
# tiles of at most 224 own rows (one consumer-group round) on the stencil configs
bash tools/gpu_r2x.sh
: > gpurun_out/r3d_summary.txt
run() {  # label args config
  timeout 300 python bench.py --config $3 --no-per-config --no-cpu-baseline --steps 300 $2 > gpurun_out/r3d.json 2> gpurun_out/r3d.err
  python -c "import json;d=json.load(open('gpurun_out/r3d.json'));print('$3 $1',round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'],d['schedule']['tiles'])" >> gpurun_out/r3d_summary.txt 2>&1 || tail -2 gpurun_out/r3d.err >> gpurun_out/r3d_summary.txt
}
for c in st27_128 lap3d_256 spin_22; do
  run "default" "" $c
  run "max_tile_rows=224" "--sched max_tile_rows=224" $c
  run "max_tile_rows=448" "--sched max_tile_rows=448" $c
done
cat gpurun_out/r3d_summary.txt
