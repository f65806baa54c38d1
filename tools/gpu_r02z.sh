#!/bin/bash
mkdir -p gpurun_out
PROBE_TAG=q64 python tools/marg_probe2.py
PROBE_TAG=q32 SAMBATEN_MARG_QB=27 python tools/marg_probe2.py
timeout 900 python -m pytest tests/test_gpu_primitives.py -q -p no:cacheprovider -k "marginals_dense" 2>&1 | tail -1
for i in 1 2; do
timeout 900 python bench.py --config C4 --steps 6 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python -c "
import json;d=json.load(open('gpurun_out/bench_c4.json'))
print('C4', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['step_ms'].items()}, d['roofline']['frac'])"
done
