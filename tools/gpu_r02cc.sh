#!/bin/bash
# persistent COO ALS: GPU suite (COO files first), C3 / C5 bench vs the per-mode pipeline
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "coo or getrank or incremental or dist" > gpurun_out/pytest_coo.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_coo.log
tail -3 gpurun_out/pytest_coo.log
FL="--steps 8 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute"
for C in C3 C5; do
  timeout 600 python bench.py --config $C $FL > gpurun_out/bench_p_$C.json 2> gpurun_out/bench_p_$C.err
  SAMBATEN_COO_ALS_MULTI=1 timeout 600 python bench.py --config $C $FL > gpurun_out/bench_m_$C.json 2> gpurun_out/bench_m_$C.err
  for V in p m; do python -c "
import json;d=json.load(open('gpurun_out/bench_${V}_$C.json'))
print('$V $C', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['step_ms'].items()}, 'fit', d.get('fit_full_last'), 'it', d.get('als_iters_per_rep'))" 2>&1 | tail -1; done
done
