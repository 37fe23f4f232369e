# session re-entry check of HEAD: GPU tests + K4/K8 timings on st27 / fem / spin
mkdir -p gpurun_out; : > gpurun_out/o_summary.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/o_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/o_tests.txt
for c in st27_128 fem_knn_4M spin_22; do
  for v in tiled_atomic tiled_colored; do
    timeout 300 python bench.py --config $c --no-per-config --no-cpu-baseline --variant $v --steps 300 > gpurun_out/o.json 2> gpurun_out/o.err
    python -c "import json;d=json.load(open('gpurun_out/o.json'));print('$c',d['variant'],round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'],d['clocks']['reasons'])" >> gpurun_out/o_summary.txt 2>&1 || tail -2 gpurun_out/o.err >> gpurun_out/o_summary.txt
  done
done
cat gpurun_out/o_summary.txt
