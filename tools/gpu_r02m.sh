#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fitinc.py tests/test_gpu_coo.py tests/test_gpu_incremental.py -q -p no:cacheprovider -x > gpurun_out/fitcoo.log 2>&1; echo "rc=$?" >> gpurun_out/fitcoo.log
FL="--steps 6 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
for c in C5 C3; do
timeout 900 python bench.py --config $c $FL > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
python -c "
import json;d=json.load(open('gpurun_out/bench_$c.json'))
print('$c', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['step_ms'].items()}, d.get('fit_full_last'), d.get('fit_path_last'))"
done
tail -n 3 gpurun_out/fitcoo.log
