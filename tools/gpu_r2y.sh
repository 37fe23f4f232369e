#!/bin/bash
# K8 signaller in the loader warp's idle lanes (default, 3 gather warps) vs a
# dedicated signaller warp (sig1.so, 2 gather warps); parity of K8 first.
mkdir -p gpurun_out; : > gpurun_out/y_summary.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "colored or full_size or powers" > gpurun_out/y_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/y_tests.txt
run() {  # label lib variant config steps
  SYMM_LIB=$2 timeout 400 python bench.py --config $4 --no-per-config --no-cpu-baseline --variant $3 --steps $5 > gpurun_out/y.json 2> gpurun_out/y.err
  python -c "import json;d=json.load(open('gpurun_out/y.json'));print('$4 $1',round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'],d.get('parity_sampled_relinf'))" >> gpurun_out/y_summary.txt 2>&1 || tail -2 gpurun_out/y.err >> gpurun_out/y_summary.txt
}
for c in st27_128 fem_knn_4M spin_22; do
  run "K8 sig2 (loader lanes)" "" tiled_colored $c 300
  run "K8 sig1 (warp)" libvariants/sig1.so tiled_colored $c 300
  run "K4" "" tiled_atomic $c 300
done
cat gpurun_out/y_summary.txt
