# K8 pipelined flush (RED in DAG order, early predecessor loads, deferred signal): parity + timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tiled_colored or full_size or small_configs or edge_cases or powers" > gpurun_out/f_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/f_tests.txt
for c in st27_128 fem_knn_4M spin_22; do
  for v in tiled_colored tiled_atomic; do
    timeout 300 python bench.py --config $c --no-per-config --variant $v --no-cpu-baseline --steps 200 > gpurun_out/f_${v}_$c.json 2> gpurun_out/f_${v}_$c.err; echo "$c $v rc=$?"
    python -c "import json;d=json.load(open('gpurun_out/f_${v}_$c.json'));print('$c',d['variant'],round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['parity_sampled_relinf'],d['clocks']['sm_mhz'])" 2>&1 | tail -1
  done
done
