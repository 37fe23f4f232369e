# Sorted tiles: free record order (SYMM_REC_FREE, default 1) and val bank-pair colouring
# (SYMM_VAL_COLOR=1): parity under the env, then A/B on fem (the config with sorted tiles)
mkdir -p gpurun_out; : > gpurun_out/r3e_summary.txt
SYMM_VAL_COLOR=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "not lap3d_512" > gpurun_out/r3e_tests.txt 2>&1; tail -3 gpurun_out/r3e_tests.txt >> gpurun_out/r3e_summary.txt
run() {  # label env variant config
  env $2 timeout 300 python bench.py --config $4 --no-per-config --no-cpu-baseline --variant $3 --steps 300 > gpurun_out/r3e.json 2> gpurun_out/r3e.err
  python -c "import json;d=json.load(open('gpurun_out/r3e.json'));print('$4 $3 $1',round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'],d.get('parity_sampled_relinf'))" >> gpurun_out/r3e_summary.txt 2>&1 || tail -2 gpurun_out/r3e.err >> gpurun_out/r3e_summary.txt
}
for rep in 1 2; do
  run "rec_free (default)" "X=1" tiled_atomic fem_knn_4M
  run "rec_free + val_color" "SYMM_VAL_COLOR=1" tiled_atomic fem_knn_4M
  run "row records first (old)" "SYMM_REC_FREE=0" tiled_atomic fem_knn_4M
done
run "rec_free (default)" "X=1" tiled_colored fem_knn_4M
run "rec_free + val_color" "SYMM_VAL_COLOR=1" tiled_colored fem_knn_4M
run "row records first (old)" "SYMM_REC_FREE=0" tiled_colored fem_knn_4M
run "rec_free (default)" "X=1" tiled fem_knn_4M
run "rec_free + val_color" "SYMM_VAL_COLOR=1" tiled fem_knn_4M
run "gain 0.1 + val_color" "SYMM_VAL_COLOR=1 SYMM_SORT_GAIN=0.1" tiled_atomic st27_128
run "gain 0.1 + val_color" "SYMM_VAL_COLOR=1 SYMM_SORT_GAIN=0.1" tiled_atomic spin_22
cat gpurun_out/r3e_summary.txt
