# usage: bash tools/gpu_ab.sh "<env settings 1>" "<env settings 2>" ...   (A/B of env knobs on the bench)
mkdir -p gpurun_out; : > gpurun_out/ab_summary.txt
for c in ${CONFIGS:-st27_128 spin_22}; do
  for e in "$@"; do
    env $e timeout 600 python bench.py --config $c --steps ${STEPS:-300} --warmup 10 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ab.json 2> gpurun_out/ab.err
    python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$c','$e',d['variant'],round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'])" >> gpurun_out/ab_summary.txt 2>&1 || tail -5 gpurun_out/ab.err >> gpurun_out/ab_summary.txt
  done
done
cat gpurun_out/ab_summary.txt
