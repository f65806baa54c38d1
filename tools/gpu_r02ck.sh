#!/bin/bash
# 128-row tiles: phases (C3, C5), COO / getrank / dist GPU tests (the rank-deficient one verbose)
mkdir -p gpurun_out
FL="--steps 3 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
for C in C3 C5; do
  SAMBATEN_COO_ALS_PROFILE=1 timeout 600 python bench.py --config $C $FL > gpurun_out/bench_pa_${C}.json 2> gpurun_out/bench_pa_${C}.err
  echo "$C"; grep coo_als_persist gpurun_out/bench_pa_${C}.err | tail -2
  python -c "
import json;d=json.load(open('gpurun_out/bench_pa_${C}.json'))
print(round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['step_ms'].items()}, 'fit', d.get('fit_full_last'))" 2>&1 | tail -1
done
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "coo or getrank or dist" > gpurun_out/pytest_coo.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_coo.log
tail -2 gpurun_out/pytest_coo.log; grep -E '^E |FAILED' gpurun_out/pytest_coo.log | head
SAMBATEN_COO_ALS_MULTI=1 timeout 600 python -m pytest tests/test_gpu_getrank.py -q -p no:cacheprovider -k "coo_rank_deficient" 2>&1 | tail -3
