# Split slots of sorted tiles (leader + partner lane, warp-shuffle combine) and
# chunk-to-warp balancing: parity, then A/B against SYMM_SPLIT=0 / SYMM_WARP_BAL=0
mkdir -p gpurun_out; : > gpurun_out/r3c_summary.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r3c_tests.txt 2>&1; tail -3 gpurun_out/r3c_tests.txt >> gpurun_out/r3c_summary.txt
run() {  # label env variant config
  env $2 timeout 300 python bench.py --config $4 --no-per-config --no-cpu-baseline --variant $3 --steps 300 > gpurun_out/r3c.json 2> gpurun_out/r3c.err
  python -c "import json;d=json.load(open('gpurun_out/r3c.json'));print('$4 $3 $1',round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'],d.get('parity_sampled_relinf'))" >> gpurun_out/r3c_summary.txt 2>&1 || tail -2 gpurun_out/r3c.err >> gpurun_out/r3c_summary.txt
}
for c in fem_knn_4M spin_22 st27_128; do
  for v in tiled_atomic tiled_colored tiled; do
    run "split+bal (default)" "X=1" $v $c
    run "no split" "SYMM_SPLIT=0" $v $c
    [ $c = fem_knn_4M ] && run "no split, no bal" "SYMM_SPLIT=0 SYMM_WARP_BAL=0" $v $c
  done
done
run "sort every tile (gain 0)" "SYMM_SORT_GAIN=0" tiled_atomic st27_128
run "sort every tile (gain 0)" "SYMM_SORT_GAIN=0" tiled_atomic spin_22
run "sort gain 0.1" "SYMM_SORT_GAIN=0.1" tiled_atomic st27_128
run "sort gain 0.1" "SYMM_SORT_GAIN=0.1" tiled_atomic spin_22
cat gpurun_out/r3c_summary.txt
