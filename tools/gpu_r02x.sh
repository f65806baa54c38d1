#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_primitives.py -q -p no:cacheprovider -k "marginals" > gpurun_out/q32.log 2>&1; echo "prim rc=$?" >> gpurun_out/q32.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider >> gpurun_out/q32.log 2>&1; echo "full rc=$?" >> gpurun_out/q32.log
timeout 900 python bench.py --config C4 --steps 6 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python -c "
import json;d=json.load(open('gpurun_out/bench_c4.json'))
print('C4', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['step_ms'].items()}, d['roofline']['frac'])"
grep -E "passed|failed|rc=" gpurun_out/q32.log
