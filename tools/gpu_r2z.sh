#!/bin/bash
# K4 tile-size sweep on the kNN (FEM-like) and spin configs with the current
# tile formats (the round-1 sweep predates the sorted record lists).
mkdir -p gpurun_out; : > gpurun_out/z_summary.txt
run() {  # config work nnz window [env]
  env $5 timeout 300 python bench.py --config $1 --no-per-config --no-cpu-baseline --steps 300 --tile-work $2 --tile-nnz $3 --tile-window $4 > gpurun_out/z.json 2> gpurun_out/z.err
  python -c "import json;d=json.load(open('gpurun_out/z.json'));print('$1 work=$2 nnz=$3 win=$4 $5',round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'],d['schedule']['tiles'])" >> gpurun_out/z_summary.txt 2>&1 || tail -2 gpurun_out/z.err >> gpurun_out/z_summary.txt
}
for c in fem_knn_4M spin_22; do
  run $c 3500 3000 1200
  run $c 2500 2200 900
  run $c 3000 2600 1000
  run $c 4200 3600 1400
  run $c 5000 4000 1600
  run $c 3500 3000 1000
  run $c 3500 3000 1500
done
run fem_knn_4M 3500 3000 1200 SYMM_SORT_GAIN=0.1
run fem_knn_4M 3500 3000 1200 SYMM_SORT_GAIN=0.5
cat gpurun_out/z_summary.txt
