#!/bin/bash
# Round evidence: default bench line, every config's bench line, the ncu launch
# list of the default bench command, and one ncu --set full capture of k_tiled.
mkdir -p gpurun_out/ev
timeout 600 python bench.py > gpurun_out/ev/bench_default.json 2> gpurun_out/ev/bench_default.err
for c in fem_knn_4M spin_22 lap3d_512; do
  timeout 900 python bench.py --config $c --steps 500 --warmup 10 > gpurun_out/ev/bench_$c.json 2> gpurun_out/ev/bench_$c.err
done
timeout 900 python bench.py --all-variants --steps 400 --no-cpu-baseline > gpurun_out/ev/bench_variants.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/ev/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tiled -c 1 -o gpurun_out/ev/k_tiled_default -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev/ncu_full.log 2>&1
ncu -i gpurun_out/ev/k_tiled_default.ncu-rep --page raw --csv > gpurun_out/ev/k_tiled_default_raw.csv 2>&1
ncu -i gpurun_out/ev/k_tiled_default.ncu-rep --page details > gpurun_out/ev/k_tiled_default_details.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tiled -c 1 -o gpurun_out/ev/k_tiled_fem -f python bench.py --config fem_knn_4M --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev/ncu_full_fem.log 2>&1
ncu -i gpurun_out/ev/k_tiled_fem.ncu-rep --page raw --csv > gpurun_out/ev/k_tiled_fem_raw.csv 2>&1
ncu -i gpurun_out/ev/k_tiled_fem.ncu-rep --page details > gpurun_out/ev/k_tiled_fem_details.txt 2>&1
