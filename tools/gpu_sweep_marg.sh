#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/sweep.txt
SBT_MARG_PC=1 timeout 600 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_incremental.py -q -p no:cacheprovider -k "marginals or incremental" > gpurun_out/pc_tests.log 2>&1; echo "pc tests rc=$?" >> gpurun_out/sweep.txt
for cfg in 0:96:192 1:96:192 1:64:192 1:48:192 1:32:192 1:48:208; do
  PC=$(echo $cfg | cut -d: -f1); S=$(echo $cfg | cut -d: -f2); Rg=$(echo $cfg | cut -d: -f3)
  SBT_MARG_PC=$PC SBT_MARG_STAGE_KB=$S SBT_MARG_RING_KB=$Rg timeout 600 python bench.py --steps 6 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute > gpurun_out/sw.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/sw.json'))
print('pc', $PC, 'stage', $S, 'ring', $Rg, 'a1', round(d['step_ms']['a1'],3), 'frac', round(d['kernels']['a1']['frac'],3), 'step', round(d['ms_per_step'],3))" >> gpurun_out/sweep.txt
done
SBT_MARG_PC=1 timeout 600 python bench.py --config C2 --steps 10 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute > gpurun_out/sw2.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/sw2.json'))
print('C2 pc a1', round(d['step_ms']['a1'],3), 'step', round(d['ms_per_step'],3))" >> gpurun_out/sweep.txt
cat gpurun_out/sweep.txt
