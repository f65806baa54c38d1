#!/bin/bash
# persistent COO ALS phase breakdown after the rows-phase fix + ncu source capture of it (C3)
mkdir -p gpurun_out
FL="--steps 2 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
for B in 2 4; do
  SAMBATEN_COO_ALS_BPS=$B SAMBATEN_COO_ALS_PROFILE=1 timeout 600 python bench.py --config C3 $FL > gpurun_out/bench_pp_C3_$B.json 2> gpurun_out/bench_pp_C3_$B.err
  echo "C3 BPS=$B"; grep coo_als_persist gpurun_out/bench_pp_C3_$B.err | tail -1
  python -c "
import json;d=json.load(open('gpurun_out/bench_pp_C3_$B.json'))
print(round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['step_ms'].items()}, 'fit', d.get('fit_full_last'))" 2>&1 | tail -1
done
FL1="--steps 1 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
SBT_PROFILE_STEP=0 timeout 900 ncu --profile-from-start off --set full --import-source on -k regex:"coo_als_persist" -c 1 \
  -o gpurun_out/prof_r02cf_c3 -f python bench.py --config C3 $FL1 > gpurun_out/ncu_r02cf.log 2>&1
echo "ncu rc=$?"
