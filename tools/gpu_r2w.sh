# gather warps: warp-cooperative 16-B cp.async per run (default) vs one bulk copy per run (bulk.so)
mkdir -p gpurun_out; : > gpurun_out/w_summary.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/w_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/w_tests.txt
run() {  # label lib variant config steps
  SYMM_LIB=$2 timeout 400 python bench.py --config $4 --no-per-config --no-cpu-baseline --variant $3 --steps $5 > gpurun_out/w.json 2> gpurun_out/w.err
  python -c "import json;d=json.load(open('gpurun_out/w.json'));print('$4 $1',round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'],d.get('parity_sampled_relinf'))" >> gpurun_out/w_summary.txt 2>&1 || tail -2 gpurun_out/w.err >> gpurun_out/w_summary.txt
}
for c in spin_22 st27_128 fem_knn_4M; do
  run "K4 coop" "" tiled_atomic $c 300
  run "K4 bulk" libvariants/bulk.so tiled_atomic $c 300
  run "K8 coop" "" tiled_colored $c 300
done
run "K4 coop" "" tiled_atomic lap3d_512 100
run "K4 bulk" libvariants/bulk.so tiled_atomic lap3d_512 100
cat gpurun_out/w_summary.txt
