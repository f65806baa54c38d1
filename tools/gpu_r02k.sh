#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_update.py tests/test_gpu_fullsize.py tests/test_gpu_edges.py -q -p no:cacheprovider -x > gpurun_out/gath.log 2>&1; echo "rc=$?" >> gpurun_out/gath.log
timeout 900 python bench.py --steps 6 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python -c "
import json;d=json.load(open('gpurun_out/bench_c4.json'))
print('C4', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['step_ms'].items()})"
tail -n 3 gpurun_out/gath.log
