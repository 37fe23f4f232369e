#!/bin/bash
mkdir -p gpurun_out
export SYMM_CS_NC=${NC:-12} SYMM_CS_WINDOW=${WW:-4096}
for sk in 1 4 5; do
SYMM_DEBUG_SKIP=$sk timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --variant colored_smem 2>&1 | tail -1 | python -c "
import sys,json
l=json.loads(sys.stdin.read()); print('skip=$sk', l.get('ms_per_step'))" >> gpurun_out/cs_decomp.txt
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_cs -c 1 -o gpurun_out/cs_prof -f python bench.py --variant colored_smem --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_cs.log 2>&1
ncu -i gpurun_out/cs_prof.ncu-rep --page details > gpurun_out/cs_prof_details.txt 2>&1
ncu -i gpurun_out/cs_prof.ncu-rep --page source --csv > gpurun_out/cs_prof_source.csv 2>&1
ncu -i gpurun_out/cs_prof.ncu-rep --page raw --csv > gpurun_out/cs_prof_raw.csv 2>&1
