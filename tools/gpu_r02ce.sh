#!/bin/bash
# persistent COO ALS phase breakdown (block 0 globaltimer per phase kind), C3 and C5
mkdir -p gpurun_out
FL="--steps 2 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
for C in C3 C5; do
for B in 2 4; do
  SAMBATEN_COO_ALS_BPS=$B SAMBATEN_COO_ALS_PROFILE=1 timeout 600 python bench.py --config $C $FL > gpurun_out/bench_pp_${C}_$B.json 2> gpurun_out/bench_pp_${C}_$B.err
  echo "$C BPS=$B"; grep coo_als_persist gpurun_out/bench_pp_${C}_$B.err | tail -2
  python -c "
import json;d=json.load(open('gpurun_out/bench_pp_${C}_$B.json'))
print(round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['step_ms'].items()}, 'fit', d.get('fit_full_last'))" 2>&1 | tail -1
done
done
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "coo" > gpurun_out/pytest_coo.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_coo.log
tail -2 gpurun_out/pytest_coo.log
