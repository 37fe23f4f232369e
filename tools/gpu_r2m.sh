# K8 immediate last-arriver signal; K4 rounds zeroed by the consumer warps (last arriver publishes)
mkdir -p gpurun_out; : > gpurun_out/m_summary.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "small_configs or edge_cases or many_tiles or full_size or powers or determin or tiled_colored" > gpurun_out/m_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/m_tests.txt
SYMM_K4_ZERO=2 SYMM_ZERO_ROUND=8 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "(small_configs or edge_cases or many_tiles or full_size) and not lap3d_512" > gpurun_out/m_tests_z2.txt 2>&1; echo "tests z2/r8 rc=$?"; tail -2 gpurun_out/m_tests_z2.txt
for c in st27_128 spin_22 fem_knn_4M; do
  for v in tiled_atomic tiled_colored; do
    timeout 300 python bench.py --config $c --no-per-config --no-cpu-baseline --variant $v --steps 300 > gpurun_out/m.json 2> gpurun_out/m.err
    python -c "import json;d=json.load(open('gpurun_out/m.json'));print('$c',d['variant'],round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'],d['clocks']['reasons'])" >> gpurun_out/m_summary.txt 2>&1 || tail -2 gpurun_out/m.err >> gpurun_out/m_summary.txt
  done
done
for e in "SYMM_K4_ZERO=0" "SYMM_K4_ZERO=2" "SYMM_K4_ZERO=2 SYMM_ZERO_ROUND=32" "SYMM_K4_ZERO=2 SYMM_ZERO_ROUND=64"; do
  env $e timeout 600 python bench.py --config lap3d_512 --no-per-config --no-cpu-baseline --steps 100 > gpurun_out/m.json 2> gpurun_out/m.err
  python -c "import json;d=json.load(open('gpurun_out/m.json'));print('lap3d_512','$e',round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'],d['clocks']['reasons'])" >> gpurun_out/m_summary.txt 2>&1 || tail -2 gpurun_out/m.err >> gpurun_out/m_summary.txt
done
cat gpurun_out/m_summary.txt
