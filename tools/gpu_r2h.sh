# K8 decomposition (K4_DEBUG_SKIP build): DAG wait / RED / flush removed in turn (diagnostics, wrong results for bits 4/16)
mkdir -p gpurun_out; : > gpurun_out/h_summary.txt
for c in st27_128 fem_knn_4M; do
  for e in "SYMM_DEBUG_SKIP=0" "SYMM_DEBUG_SKIP=64" "SYMM_DEBUG_SKIP=16" "SYMM_DEBUG_SKIP=80" "SYMM_DEBUG_SKIP=112" "SYMM_DEBUG_SKIP=4" "SYMM_DEBUG_SKIP=84"; do
    env SYMM_LIB=libvariants/dbg.so $e timeout 300 python bench.py --config $c --no-per-config --variant tiled_colored --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/h.json 2> gpurun_out/h.err
    python -c "import json;d=json.load(open('gpurun_out/h.json'));print('$c','$e',d['variant'],round(d['ms_per_step'],4),d['clocks']['sm_mhz'])" >> gpurun_out/h_summary.txt 2>&1 || tail -3 gpurun_out/h.err >> gpurun_out/h_summary.txt
  done
  env SYMM_LIB=libvariants/dbg.so timeout 300 python bench.py --config $c --no-per-config --variant tiled_atomic --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/h.json 2> gpurun_out/h.err
  python -c "import json;d=json.load(open('gpurun_out/h.json'));print('$c','K4 dbg build',d['variant'],round(d['ms_per_step'],4),d['clocks']['sm_mhz'])" >> gpurun_out/h_summary.txt 2>&1
done
cat gpurun_out/h_summary.txt
