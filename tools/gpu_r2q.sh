# K8 decomposition with the signaller (debug-skip build: 4 no flush, 16 no DAG wait)
mkdir -p gpurun_out; : > gpurun_out/q_summary.txt
for c in st27_128 spin_22; do
  for s in 0 16 4 20; do
    SYMM_LIB=libvariants/dbg.so SYMM_DEBUG_SKIP=$s timeout 300 python bench.py --config $c --no-per-config --no-cpu-baseline --variant tiled_colored --steps 300 > gpurun_out/q.json 2> gpurun_out/q.err
    python -c "import json;d=json.load(open('gpurun_out/q.json'));print('$c K8 dbg skip=$s',round(d['ms_per_step'],4),d['clocks']['sm_mhz'])" >> gpurun_out/q_summary.txt 2>&1 || tail -2 gpurun_out/q.err >> gpurun_out/q_summary.txt
  done
  SYMM_LIB=libvariants/dbg.so timeout 300 python bench.py --config $c --no-per-config --no-cpu-baseline --variant tiled_atomic --steps 300 > gpurun_out/q.json 2> gpurun_out/q.err
  python -c "import json;d=json.load(open('gpurun_out/q.json'));print('$c K4 dbg build',round(d['ms_per_step'],4),d['clocks']['sm_mhz'])" >> gpurun_out/q_summary.txt 2>&1
done
cat gpurun_out/q_summary.txt
