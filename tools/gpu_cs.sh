#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/cs_bench.txt
timeout 300 python tools/cs_check.py colored_smem 2>&1 | grep -v "^Exception\|^Traceback\|^  File\|^TypeError" > gpurun_out/cs_check.txt
for cfg in ${CFGS:-12:4096:16384:0}; do
  IFS=: read -r c1 c2 c3 c4 c5 <<< "$cfg"; set -- $c1 $c2 $c3 $c4 ${c5:-4}
  SYMM_CS_NC=$1 SYMM_CS_WINDOW=$2 SYMM_CS_CHUNK=$3 SYMM_DEBUG_SKIP=$4 SYMM_CS_V=$5 timeout 300 python bench.py --config ${CFG:-st27_128} --steps 300 --warmup 10 --no-cpu-baseline --variant colored_smem 2>&1 | tail -1 | python -c "
import sys,json
t=sys.stdin.read()
try:
  l=json.loads(t); print('NC=$1 W=$2 CH=$3 skip=$4 V=$5', l.get('ms_per_step'), l.get('roofline',{}).get('frac'), l.get('error'))
except Exception: print('NC=$1 W=$2 CH=$3 FAILED', t[-300:])" >> gpurun_out/cs_bench.txt 2>&1
done
