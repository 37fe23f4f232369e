# usage: bash tools/gpu_r2.sh <tag> [pytest-args...]   (round-2 generic: tests + bench lines)
tag=$1; shift
mkdir -p gpurun_out
if [ "$1" != "--no-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/${tag}_tests.txt 2>&1; echo "tests rc=$?"
  tail -3 gpurun_out/${tag}_tests.txt
fi
for c in ${CONFIGS:-st27_128 fem_knn_4M spin_22}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-300} --warmup 10 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/${tag}_$c.json 2> gpurun_out/${tag}_$c.err; echo "$c rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/${tag}_$c.json'));print('$c',d['variant'],round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks'])" 2>/dev/null
done
