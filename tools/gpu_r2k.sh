# A/B: HEAD lib vs lane-0 loader vs current (K4 on st27/spin/fem); lap3d zero modes + ncu DRAM bytes; K8 decomposition
mkdir -p gpurun_out; : > gpurun_out/k_summary.txt
for c in st27_128 spin_22 fem_knn_4M; do
  for lib in libvariants/head.so libvariants/lane0.so paper_1907_06487_b200/libsymmspmv.so; do
    SYMM_LIB=$lib timeout 300 python bench.py --config $c --no-per-config --no-cpu-baseline --steps 300 > gpurun_out/k.json 2> gpurun_out/k.err
    python -c "import json;d=json.load(open('gpurun_out/k.json'));print('$c','$lib',d['variant'],round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'],d['clocks']['reasons'])" >> gpurun_out/k_summary.txt 2>&1 || tail -2 gpurun_out/k.err >> gpurun_out/k_summary.txt
  done
done
for e in "SYMM_LIB=libvariants/head.so" "SYMM_K4_ZERO=0" "SYMM_K4_ZERO=2"; do
  env $e timeout 600 python bench.py --config lap3d_512 --no-per-config --no-cpu-baseline --steps 100 > gpurun_out/k.json 2> gpurun_out/k.err
  python -c "import json;d=json.load(open('gpurun_out/k.json'));print('lap3d_512','$e',round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'],d['clocks']['reasons'])" >> gpurun_out/k_summary.txt 2>&1 || tail -2 gpurun_out/k.err >> gpurun_out/k_summary.txt
done
cat gpurun_out/k_summary.txt
for z in 0 2; do
  SYMM_K4_ZERO=$z timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum --clock-control none -k regex:"k_tiled|k_zero" -c 6 --csv python tools/run_n.py lap3d_512 tiled_atomic 3 > gpurun_out/k_ncu_lap_z$z.csv 2>&1; echo "ncu z$z rc=$?"
done
: > gpurun_out/h_summary.txt
for e in "SYMM_DEBUG_SKIP=0" "SYMM_DEBUG_SKIP=64" "SYMM_DEBUG_SKIP=16" "SYMM_DEBUG_SKIP=80" "SYMM_DEBUG_SKIP=4" "SYMM_DEBUG_SKIP=84"; do
  env SYMM_LIB=libvariants/dbg.so $e timeout 300 python bench.py --config st27_128 --no-per-config --variant tiled_colored --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/h.json 2> gpurun_out/h.err
  python -c "import json;d=json.load(open('gpurun_out/h.json'));print('st27 K8 dbg','$e',round(d['ms_per_step'],4),d['clocks']['sm_mhz'])" >> gpurun_out/h_summary.txt 2>&1 || tail -3 gpurun_out/h.err >> gpurun_out/h_summary.txt
done
cat gpurun_out/h_summary.txt
