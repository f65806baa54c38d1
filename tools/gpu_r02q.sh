#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_coo.py tests/test_gpu_incremental.py tests/test_gpu_dist.py tests/test_gpu_getrank.py tests/test_gpu_fitinc.py tests/test_gpu_recompute.py -q -p no:cacheprovider -x > gpurun_out/coo_als.log 2>&1; echo "rc=$?" >> gpurun_out/coo_als.log
FL="--steps 6 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
for c in "C5 config" "C3 config" "C5 cold"; do
set -- $c
timeout 900 python bench.py --config $1 --als-init $2 $FL > gpurun_out/bench_$1_$2.json 2> gpurun_out/bench_$1_$2.err
python -c "
import json;d=json.load(open('gpurun_out/bench_$1_$2.json'))
print('$c', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['step_ms'].items()}, d.get('fit_full_last'), d.get('als_iters_per_rep'))"
done
tail -n 3 gpurun_out/coo_als.log
