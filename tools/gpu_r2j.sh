# (1) flush targets out of the copied block (gather warp expands runs); (2) K4 y zeroing in rounds by the loader warp
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "small_configs or edge_cases or many_tiles or eigen or full_size or powers or multirank or determin" > gpurun_out/j_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/j_tests.txt
SYMM_K4_ZERO=2 SYMM_ZERO_ROUND=8 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "(small_configs or edge_cases or many_tiles or full_size) and not lap3d_512" > gpurun_out/j_tests_z2.txt 2>&1; echo "tests z2/r8 rc=$?"; tail -2 gpurun_out/j_tests_z2.txt
for e in "SYMM_K4_ZERO=2" "SYMM_K4_ZERO=0" "SYMM_K4_ZERO=2 SYMM_ZERO_ROUND=32"; do
  env $e timeout 600 python bench.py --config lap3d_512 --no-per-config --cpu-seconds 2 --steps 100 > gpurun_out/j.json 2> gpurun_out/j.err; echo "lap $e rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/j.json'));print('lap3d_512','$e',round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['parity_sampled_relinf'],d['clocks']['sm_mhz'],d['clocks']['reasons'])" 2>&1 | tail -1
done
for c in st27_128 spin_22 fem_knn_4M; do
  for e in "SYMM_TGT_IN_BLOCK=0" "SYMM_TGT_IN_BLOCK=1"; do
    env $e timeout 600 python bench.py --config $c --no-per-config --no-cpu-baseline --steps 200 > gpurun_out/j.json 2> gpurun_out/j.err; echo "$c $e rc=$?"
    python -c "import json;d=json.load(open('gpurun_out/j.json'));print('$c','$e',d['variant'],round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'],d['clocks']['reasons'])" 2>&1 | tail -1
  done
done
