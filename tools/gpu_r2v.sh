# gather-warp count: K4 with 2 gather warps (g2.so) vs 3; K8 without the signaller (3 gather warps, nosig.so)
mkdir -p gpurun_out; : > gpurun_out/v_summary.txt
run() {  # label lib variant config
  SYMM_LIB=$2 timeout 300 python bench.py --config $4 --no-per-config --no-cpu-baseline --variant $3 --steps 300 > gpurun_out/v.json 2> gpurun_out/v.err
  python -c "import json;d=json.load(open('gpurun_out/v.json'));print('$4 $1',round(d['ms_per_step'],4),d['clocks']['sm_mhz'],d.get('parity_sampled_relinf'))" >> gpurun_out/v_summary.txt 2>&1 || tail -2 gpurun_out/v.err >> gpurun_out/v_summary.txt
}
for c in spin_22 st27_128 fem_knn_4M; do
  run "K4 3 gather" "" tiled_atomic $c
  run "K4 2 gather" libvariants/g2.so tiled_atomic $c
  run "K8 signaller (2 gather)" "" tiled_colored $c
  run "K8 no signaller (3 gather)" libvariants/nosig.so tiled_colored $c
done
cat gpurun_out/v_summary.txt
