# K8 with per-position metadata prefetched a group tile ahead (acquire loads before the stage waits)
mkdir -p gpurun_out; : > gpurun_out/u_summary.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "colored or full_size or powers" > gpurun_out/u_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/u_tests.txt
for c in st27_128 fem_knn_4M spin_22; do
  for v in tiled_colored tiled_atomic; do
    timeout 300 python bench.py --config $c --no-per-config --no-cpu-baseline --variant $v --steps 300 > gpurun_out/u.json 2> gpurun_out/u.err
    python -c "import json;d=json.load(open('gpurun_out/u.json'));print('$c',d['variant'],round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'])" >> gpurun_out/u_summary.txt 2>&1 || tail -2 gpurun_out/u.err >> gpurun_out/u_summary.txt
  done
done
cat gpurun_out/u_summary.txt
