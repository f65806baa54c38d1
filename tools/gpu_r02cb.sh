#!/bin/bash
# ncu --set full of the C3 COO ALS kernels (one timed step; first iteration's launches)
TAG=r02cb
mkdir -p gpurun_out
FL="--steps 1 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
SBT_PROFILE_STEP=0 timeout 1200 ncu --profile-from-start off --set full --import-source on \
  -k regex:"coo_mttkrp_piece|als_rows_kernel|als_scale|als_reduce|als_vinv|coo_piece_fixup" -c 18 \
  -o gpurun_out/prof_${TAG}_c3 -f python bench.py --config C3 $FL > gpurun_out/ncu_${TAG}_c3.log 2>&1
echo "c3 rc=$?"
python - <<'PY' > gpurun_out/c3_shapes.txt 2>&1
import numpy as np, sys
sys.path.insert(0,'.')
PY
