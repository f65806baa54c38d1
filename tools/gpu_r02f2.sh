#!/bin/bash
# DRAM traffic per launch of the step kernels (single-pass metrics: no kernel replay of the 108 GB store)
mkdir -p gpurun_out
FL1="--steps 1 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
for C in C4 C2 C3 C5; do
SBT_PROFILE_STEP=0 timeout 900 ncu --profile-from-start off --metrics $M --clock-control none --csv \
    --log-file gpurun_out/traffic_r02f_$C.csv python bench.py --config $C $FL1 > /dev/null 2>&1
echo "$C rc=$?"
done
