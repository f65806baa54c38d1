#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/sw.txt
for cfg in "0 0 96 192" "1 0 96 192" "0 8 96 192" "1 8 96 192" "1 0 72 216" "0 0 104 208"; do
  set -- $cfg
  SBT_MARG_PC=$1 SBT_MARG_NCH=$2 SBT_MARG_STAGE_KB=$3 SBT_MARG_RING_KB=$4 timeout 600 python bench.py --config C4 --steps 6 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute > gpurun_out/sw.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/sw.json'))
print('$cfg', 'a1', round(d['step_ms']['a1'],3), 'frac', round(d['kernels']['a1']['frac'],3))" >> gpurun_out/sw.txt
done
cat gpurun_out/sw.txt
