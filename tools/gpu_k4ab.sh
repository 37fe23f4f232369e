#!/bin/bash
# K4 A/B: bank-aware entry order on/off, several configs
mkdir -p gpurun_out; rm -f gpurun_out/k4ab.txt
python tools/cs_check.py tiled_atomic 2>&1 | grep tiled >> gpurun_out/k4ab.txt
python tools/cs_check.py tiled 2>&1 | grep tiled >> gpurun_out/k4ab.txt
for c in ${CFGS:-st27_128 fem_knn_4M spin_22 lap3d_256}; do
 for nb in ""; do
  SYMM_NO_BANK_ORDER=$nb timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline --variant tiled_atomic 2>&1 | tail -1 | python -c "
import sys,json
l=json.loads(sys.stdin.read()); print('$c nobank=$nb', l['ms_per_step'], l['roofline']['frac'])" >> gpurun_out/k4ab.txt
 done
done
