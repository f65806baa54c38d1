#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_coo.py tests/test_gpu_getrank.py tests/test_gpu_dist.py tests/test_gpu_fitinc.py tests/test_gpu_incremental.py -q -p no:cacheprovider > gpurun_out/af.log 2>&1; echo "rc=$?" >> gpurun_out/af.log
tail -n 2 gpurun_out/af.log
for c in C5 C3; do
timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute > gpurun_out/b.json 2> gpurun_out/b.err
python -c "
import json;d=json.load(open('gpurun_out/b.json'))
print('$c', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['step_ms'].items()}, repr(d['fit_full_last']))"
done
SBT_PROFILE_STEP=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_af_c5.csv python bench.py --config C5 --steps 1 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute > /dev/null 2>&1
