#!/bin/bash
mkdir -p gpurun_out
FL1="--steps 1 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
SBT_PROFILE_STEP=0 timeout 900 ncu --profile-from-start off --set full --import-source on -k regex:"coo_als_persist" -c 1 \
  -o gpurun_out/prof_r02cl_c3 -f python bench.py --config C3 $FL1 > gpurun_out/ncu_r02cl.log 2>&1
echo "ncu rc=$?"
