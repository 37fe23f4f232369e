#!/bin/bash
# work-sorted lane positions: SYMM_SORT_GAIN sweep on several configs (tiled_atomic), + parity tests of the tiled variants
mkdir -p gpurun_out; rm -f gpurun_out/sort.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "tiled" > gpurun_out/sort_pytest.txt 2>&1; tail -2 gpurun_out/sort_pytest.txt >> gpurun_out/sort.txt
for cfg in ${CFGS:-st27_128 fem_knn_4M spin_22}; do
  for g in ${GAINS:-1 0.1 0}; do
    SYMM_SORT_GAIN=$g timeout 400 python bench.py --config $cfg --steps 300 --warmup 10 --no-cpu-baseline --variant ${VARIANT:-tiled_atomic} 2>&1 | tail -1 | python -c "
import sys,json
t=sys.stdin.read()
try:
  l=json.loads(t); print('$cfg gain=$g', round(l['ms_per_step'],4), round(l['roofline']['frac'],3), l['schedule']['plan'])
except Exception: print('$cfg gain=$g FAILED', t[-300:])" >> gpurun_out/sort.txt 2>&1
  done
done
cat gpurun_out/sort.txt
