#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/nch.txt
for n in 0 8 16; do
  SBT_MARG_NCH=$n timeout 900 python bench.py --config C4 --steps 6 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute > gpurun_out/nch.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/nch.json'))
print('nch', $n, 'a1', round(d['step_ms']['a1'],3), 'frac', round(d['kernels']['a1']['frac'],3), 'step', round(d['ms_per_step'],3))" >> gpurun_out/nch.txt
done
SBT_MARG_NCH=8 timeout 600 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "marginals or c4" >> gpurun_out/nch.txt 2>&1
cat gpurun_out/nch.txt | tail -6
