# A/B: L2 prefetch of tile blocks (loader, bit 0) and of the x window (gather
# warps, bit 1), alone and combined with fewer / larger consumer groups
mkdir -p gpurun_out; : > gpurun_out/u_summary.txt
run() {  # label lib variant config
  SYMM_LIB=$2 timeout 300 python bench.py --config $4 --no-per-config --no-cpu-baseline --variant $3 --steps 300 > gpurun_out/u.json 2> gpurun_out/u.err
  python -c "import json;d=json.load(open('gpurun_out/u.json'));print('$4 $3 $1',round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'],d.get('parity_sampled_relinf'))" >> gpurun_out/u_summary.txt 2>&1 || tail -2 gpurun_out/u.err >> gpurun_out/u_summary.txt
}
for c in ${CFGS:-fem_knn_4M spin_22 st27_128 lap3d_256}; do
  for l in ${LIBS:-default pf1 pf2 pf3 g2x14 g2x14pf3 g3x9pf3}; do
    lib=libvariants/$l.so; [ $l = default ] && lib=""
    run "$l" "$lib" tiled_atomic $c
  done
  run "default" "" tiled_colored $c
  run "pf3" libvariants/pf3.so tiled_colored $c
done
cat gpurun_out/u_summary.txt
