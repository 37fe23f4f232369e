#!/bin/bash
# Single-run tiles without tgt[] (TileDesc.gather_runs bit 1): GPU tests, smoke, A/B on the
# stencil configs against SYMM_SINGLE_RUN=0, then the default bench line
mkdir -p gpurun_out/g; : > gpurun_out/g/summary.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g/gputests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/g/summary.txt; tail -2 gpurun_out/g/gputests.txt >> gpurun_out/g/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/g/summary.txt
run() {  # label env variant config
  env $2 timeout 600 python bench.py --config $4 --no-per-config --no-cpu-baseline --variant $3 --steps 200 > gpurun_out/g/r.json 2> gpurun_out/g/r.err
  python -c "import json;d=json.load(open('gpurun_out/g/r.json'));print('$4 $3 $1',round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'],d['schedule']['device_bytes'])" >> gpurun_out/g/summary.txt 2>&1 || tail -2 gpurun_out/g/r.err >> gpurun_out/g/summary.txt
}
for c in lap3d_256 lap3d_512; do
  for rep in 1 2; do
    run "single-run (default)" "X=1" tiled_atomic $c
    run "tgt[] in every block" "SYMM_SINGLE_RUN=0" tiled_atomic $c
  done
done
run "single-run (default)" "X=1" tiled_colored lap3d_256
run "tgt[] in every block" "SYMM_SINGLE_RUN=0" tiled_colored lap3d_256
run "single-run (default)" "X=1" tiled lap3d_256
run "tgt[] in every block" "SYMM_SINGLE_RUN=0" tiled lap3d_256
run "single-run (default)" "X=1" tiled_atomic st27_128
run "tgt[] in every block" "SYMM_SINGLE_RUN=0" tiled_atomic st27_128
cat gpurun_out/g/summary.txt
timeout 900 python bench.py > gpurun_out/g/bench_default.json 2> gpurun_out/g/bench_default.err; echo "bench rc=$?"
