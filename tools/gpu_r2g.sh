# K4 streamed y zeroing (large y): parity with the mode forced on small configs, full-size lap3d_512, A/B timing
mkdir -p gpurun_out
SYMM_K4_ZERO=2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "(small_configs or edge_cases or many_tiles or eigen) and tiled_atomic" > gpurun_out/g_tests_z2.txt 2>&1; echo "tests z2 rc=$?"; tail -3 gpurun_out/g_tests_z2.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "full_size and lap3d" > gpurun_out/g_tests_full.txt 2>&1; echo "tests full rc=$?"; tail -3 gpurun_out/g_tests_full.txt
for z in 2 0; do
  SYMM_K4_ZERO=$z timeout 600 python bench.py --config lap3d_512 --no-per-config --cpu-seconds 2 --steps 100 > gpurun_out/g_lap_z$z.json 2> gpurun_out/g_lap_z$z.err; echo "lap z=$z rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/g_lap_z$z.json'));print('z$z',d['variant'],round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['parity_sampled_relinf'],d['clocks']['sm_mhz'],d['clocks']['reasons'])" 2>&1 | tail -1
done
for z in 2 1; do
  SYMM_K4_ZERO=$z timeout 300 python bench.py --config st27_128 --no-per-config --no-cpu-baseline --steps 200 > gpurun_out/g_st27_z$z.json 2> gpurun_out/g_st27_z$z.err; echo "st27 z=$z rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/g_st27_z$z.json'));print('z$z',d['variant'],round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['parity_sampled_relinf'],d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
