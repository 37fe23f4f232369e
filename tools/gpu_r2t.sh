# ncu --set full (+source) of K8 and K4 on spin_22
mkdir -p gpurun_out/t
for v in tiled_colored tiled_atomic; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tiled -c 1 -o gpurun_out/t/${v}_spin -f python bench.py --config spin_22 --variant $v --steps 3 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/t/${v}.log 2>&1
  ncu -i gpurun_out/t/${v}_spin.ncu-rep --page source --csv > gpurun_out/t/${v}_source.csv 2>&1
  ncu -i gpurun_out/t/${v}_spin.ncu-rep --page details > gpurun_out/t/${v}_details.txt 2>&1
  ncu -i gpurun_out/t/${v}_spin.ncu-rep --page raw --csv > gpurun_out/t/${v}_raw.csv 2>&1
done
ls -la gpurun_out/t
