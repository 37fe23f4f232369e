#!/bin/bash
# A/B of alternative library builds in libvariants/*.so (compile-time kernel shapes)
mkdir -p gpurun_out; rm -f gpurun_out/libab.txt
cp paper_1907_06487_b200/libsymmspmv.so /tmp/lib_default.so
for lib in /tmp/lib_default.so libvariants/*.so; do
  cp $lib paper_1907_06487_b200/libsymmspmv.so
  for c in ${CFGS:-st27_128 lap3d_256 fem_knn_4M}; do
    timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu-baseline --variant ${VARIANT:-tiled_atomic} 2>&1 | tail -1 | python -c "
import sys,json
t=sys.stdin.read()
try:
  l=json.loads(t); print('$(basename $lib) $c', l['ms_per_step'], l['roofline']['frac'], l['schedule']['plan'].get('tiled_stages'))
except Exception: print('$(basename $lib) $c FAILED', t[-200:])" >> gpurun_out/libab.txt
  done
done
cp /tmp/lib_default.so paper_1907_06487_b200/libsymmspmv.so
