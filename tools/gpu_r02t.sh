#!/bin/bash
mkdir -p gpurun_out
SBT_PROFILE_STEP=0 timeout 1200 ncu --profile-from-start off --set full --import-source on -k regex:"coo_gather|marg_coo_rep|coo_mttkrp" -c 6 -o gpurun_out/prof_r02_c5 python bench.py --config C5 --steps 1 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute > gpurun_out/ncu_c5.log 2>&1
echo rc=$?
