# K8 base-pipeline diagnostics: acquire-load cost (acq2 = relaxed, no fence: diagnostics),
# no flush / no wait (dbg skip bits), and K4 run in K8's phase-major tile order
mkdir -p gpurun_out; : > gpurun_out/s_summary.txt
run() {  # label lib skip variant config
  SYMM_LIB=$2 SYMM_DEBUG_SKIP=$3 timeout 300 python bench.py --config $5 --no-per-config --no-cpu-baseline --variant $4 --steps 300 > gpurun_out/s.json 2> gpurun_out/s.err
  python -c "import json;d=json.load(open('gpurun_out/s.json'));print('$5 $1',round(d['ms_per_step'],4),d['clocks']['sm_mhz'])" >> gpurun_out/s_summary.txt 2>&1 || tail -2 gpurun_out/s.err >> gpurun_out/s_summary.txt
}
for c in spin_22 st27_128; do
  run "K8 default" "" 0 tiled_colored $c
  run "K8 acq2 (relaxed, diag)" libvariants/acq2.so 0 tiled_colored $c
  run "K8 dbg skip16 (no wait)" libvariants/dbg.so 16 tiled_colored $c
  run "K8 dbg skip20 (no wait/flush)" libvariants/dbg.so 20 tiled_colored $c
  run "K4 default" "" 0 tiled_atomic $c
  run "K4 phase-major order" libvariants/k4order.so 0 tiled_atomic $c
done
cat gpurun_out/s_summary.txt
