#!/bin/bash
mkdir -p gpurun_out
for cfg in 96:192 64:192 48:192 48:216 32:192 72:216; do
  S=${cfg%%:*}; Rg=${cfg##*:}
  SBT_MARG_STAGE_KB=$S SBT_MARG_RING_KB=$Rg timeout 600 python bench.py --steps 6 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute > gpurun_out/sweep_$S_$Rg.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/sweep_$S_$Rg.json'))
print('stage', $S, 'ring', $Rg, 'a1', round(d['step_ms']['a1'],3), 'frac', round(d['kernels']['a1']['frac'],3), 'step', round(d['ms_per_step'],3))" >> gpurun_out/sweep.txt
done
cat gpurun_out/sweep.txt
