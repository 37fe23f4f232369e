# K4 zeroing in rounds (large y) + K8 with equitable phases: parity, A/B timings
mkdir -p gpurun_out
SYMM_K4_ZERO=2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "(small_configs or edge_cases or many_tiles or eigen) and tiled_atomic" > gpurun_out/i_tests_z2.txt 2>&1; echo "tests z2 rc=$?"; tail -2 gpurun_out/i_tests_z2.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "full_size or tiled_colored" > gpurun_out/i_tests_full.txt 2>&1; echo "tests full rc=$?"; tail -2 gpurun_out/i_tests_full.txt
for z in 2 0; do
  SYMM_K4_ZERO=$z timeout 600 python bench.py --config lap3d_512 --no-per-config --cpu-seconds 2 --steps 100 > gpurun_out/i_lap_z$z.json 2> gpurun_out/i_lap_z$z.err; echo "lap z=$z rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/i_lap_z$z.json'));print('z$z',d['variant'],round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['parity_sampled_relinf'],d['clocks']['sm_mhz'],d['clocks']['reasons'])" 2>&1 | tail -1
done
for c in st27_128 fem_knn_4M spin_22; do
  for v in tiled_atomic tiled_colored; do
    timeout 300 python bench.py --config $c --no-per-config --variant $v --no-cpu-baseline --steps 200 > gpurun_out/i_${v}_$c.json 2> gpurun_out/i_${v}_$c.err; echo "$c $v rc=$?"
    python -c "import json;d=json.load(open('gpurun_out/i_${v}_$c.json'));print('$c',d['variant'],round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'])" 2>&1 | tail -1
  done
done
