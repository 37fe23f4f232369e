set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; grep -m1 "model name" /proc/cpuinfo; free -g
for c in st27_128 fem_knn_4M spin_22 lap3d_512; do
  timeout 600 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/base_$c.json 2> gpurun_out/base_$c.err; echo "$c rc=$?"
done
