#!/bin/bash
# Round-2 final captures: C4p stand-in (a1 with the 32-bit kernel C4 runs, a3 slice-ordered gather,
# a4 grid plan, a7 fitrows), C5 COO kernels, launch lists of one timed C4 and C5 step.
TAG=r02b
mkdir -p gpurun_out
CMDP="python bench.py --config C4p --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-variant --no-getrank --no-recompute"
for KS in marg_stream:3 gather_dense:2 als_cluster:2 fitrows:8; do
  KN=${KS%%:*}; SK=${KS##*:}
  SBT_MARG_FORCE_QB=27 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$KN -s $SK -c 1 \
      -o gpurun_out/prof_${TAG}_c4p_$KN -f $CMDP > gpurun_out/ncu_${TAG}_c4p_$KN.log 2>&1
  echo "$KN rc=$?"
done
FL="--steps 1 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
SBT_PROFILE_STEP=0 timeout 1500 ncu --profile-from-start off --set full --import-source on -k regex:"coo_gather|marg_coo_rep|coo_mttkrp|radix_scatter|permute3" -c 8 -o gpurun_out/prof_${TAG}_c5 -f python bench.py --config C5 $FL > gpurun_out/ncu_${TAG}_c5.log 2>&1
echo "c5 rc=$?"
SBT_PROFILE_STEP=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}_c4.csv python bench.py --config C4 $FL > /dev/null 2>&1
echo "c4 launches rc=$?"
SBT_PROFILE_STEP=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}_c5.csv python bench.py --config C5 $FL > /dev/null 2>&1
echo "c5 launches rc=$?"
