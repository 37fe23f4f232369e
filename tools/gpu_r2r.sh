# K8: table pointers in shared memory, first-writer flags loaded before the sums,
# predecessor counters loaded relaxed + one acquire fence before the flush (K8_ACQ=1)
# vs acquire loads (K8_ACQ=0, libvariants/acq0.so)
mkdir -p gpurun_out; : > gpurun_out/r_summary.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "colored or full_size or powers" > gpurun_out/r_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r_tests.txt
for c in st27_128 fem_knn_4M spin_22; do
  for L in "" libvariants/acq0.so; do
    SYMM_LIB=$L timeout 300 python bench.py --config $c --no-per-config --no-cpu-baseline --variant tiled_colored --steps 300 > gpurun_out/r.json 2> gpurun_out/r.err
    python -c "import json;d=json.load(open('gpurun_out/r.json'));print('$c K8 lib=$L',round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'])" >> gpurun_out/r_summary.txt 2>&1 || tail -2 gpurun_out/r.err >> gpurun_out/r_summary.txt
  done
done
cat gpurun_out/r_summary.txt
