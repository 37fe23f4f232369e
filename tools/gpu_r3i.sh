#!/bin/bash
# Tile-size sweep on the stencil configs with single-run tiles (bigger tiles: fewer spill slots per row)
mkdir -p gpurun_out; : > gpurun_out/r3i_summary.txt
run() {  # label args config
  timeout 600 python bench.py --config $3 --no-per-config --no-cpu-baseline --steps 200 $2 > gpurun_out/r3i.json 2> gpurun_out/r3i.err
  python -c "import json;d=json.load(open('gpurun_out/r3i.json'));print('$3 $1',round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'],d['schedule']['tiles'],d['schedule']['device_bytes'],d.get('parity_sampled_relinf'))" >> gpurun_out/r3i_summary.txt 2>&1 || tail -2 gpurun_out/r3i.err >> gpurun_out/r3i_summary.txt
}
for c in lap3d_256 lap3d_512; do
  run "default (3500/3000/1200)" "" $c
  run "work 3000" "--tile-work 3000" $c
  run "work 4500 window 1500" "--tile-work 4500 --tile-nnz 3500 --tile-window 1500" $c
  run "work 5500 window 1800" "--tile-work 5500 --tile-nnz 4000 --tile-window 1800" $c
  run "work 6900 window 1790" "--tile-work 6900 --tile-nnz 5000 --tile-window 1790" $c
  run "default (3500/3000/1200)" "" $c
done
cat gpurun_out/r3i_summary.txt
