# K8 signaller warp: parity (all tests touching tiled_colored) + timings
mkdir -p gpurun_out; : > gpurun_out/p_summary.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "colored or full_size or powers" > gpurun_out/p_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/p_tests.txt
for c in st27_128 fem_knn_4M spin_22; do
  for v in tiled_colored; do
    timeout 300 python bench.py --config $c --no-per-config --no-cpu-baseline --variant $v --steps 300 > gpurun_out/p.json 2> gpurun_out/p.err
    python -c "import json;d=json.load(open('gpurun_out/p.json'));print('$c',d['variant'],round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'],d['clocks']['reasons'],d.get('parity_sampled_relinf'))" >> gpurun_out/p_summary.txt 2>&1 || tail -2 gpurun_out/p.err >> gpurun_out/p_summary.txt
  done
done
cat gpurun_out/p_summary.txt
