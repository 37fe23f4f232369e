#!/bin/bash
# GPU-box script: microbenchmarks + k_tiled pipeline decomposition (debug skip bits:
# 1 row pass, 2 CSC pass, 4 flush, 8 spill gather).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 120 ./tools/micro > gpurun_out/micro.txt 2>&1
CFG=${CFG:-st27_128}
for s in 0 1 2 3 4 8 15; do
  SYMM_DEBUG_SKIP=$s timeout 300 python bench.py --config $CFG --steps 300 --warmup 10 --no-cpu-baseline --variant tiled_atomic 2>&1 | tail -1 | python -c "
import sys,json
l=json.loads(sys.stdin.read()); print('skip=$s', l['ms_per_step'], l['roofline']['frac'])" >> gpurun_out/decomp.txt
done
