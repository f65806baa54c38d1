#!/bin/bash
# persistent COO ALS: per-block barrier arrival spread (C3, C5)
mkdir -p gpurun_out
FL="--steps 2 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
for C in C3 C5; do
  SAMBATEN_COO_ALS_BPS=4 SAMBATEN_COO_ALS_PROFILE=1 timeout 600 python bench.py --config $C $FL > gpurun_out/bench_pa_${C}.json 2> gpurun_out/bench_pa_${C}.err
  echo "$C"; grep coo_als_persist gpurun_out/bench_pa_${C}.err | tail -2
done
