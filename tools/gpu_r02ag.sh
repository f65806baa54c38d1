#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_update.py tests/test_gpu_edges.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q -p no:cacheprovider > gpurun_out/ag.log 2>&1; echo "rc=$?" >> gpurun_out/ag.log
tail -n 2 gpurun_out/ag.log
timeout 900 python bench.py --config C4 --steps 10 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute > gpurun_out/b.json 2> gpurun_out/b.err
python -c "
import json;d=json.load(open('gpurun_out/b.json'))
print('C4', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['step_ms'].items()}, repr(d['fit_full_last']))"
