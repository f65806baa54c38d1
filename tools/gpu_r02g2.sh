#!/bin/bash
mkdir -p gpurun_out
FL="--steps 2 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
SAMBATEN_COO_ALS_PROFILE=1 timeout 600 python bench.py --config C3 $FL > gpurun_out/bench_pa_C3.json 2> gpurun_out/bench_pa_C3.err
grep coo_als_persist gpurun_out/bench_pa_C3.err | tail -3
