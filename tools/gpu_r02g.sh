#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_edges.py -q -p no:cacheprovider -k "grid or rank32 or zeroed" > gpurun_out/grid.log 2>&1; echo "rc=$?" >> gpurun_out/grid.log
for G in 0 1; do
  SAMBATEN_ALS_GRID=$G timeout 900 python bench.py --config C2 --steps 20 --warmup 5 --no-getrank --no-variant --no-cpu-baseline --no-recompute --no-e2e > gpurun_out/bench_c2_g$G.json 2> gpurun_out/bench_c2_g$G.err
  SAMBATEN_ALS_GRID=$G timeout 900 python bench.py --steps 6 --warmup 3 --no-getrank --no-cpu-baseline --no-recompute --no-e2e --als-init cold > gpurun_out/bench_c4cold_g$G.json 2> gpurun_out/bench_c4cold_g$G.err
  SAMBATEN_ALS_GRID=$G timeout 900 python bench.py --steps 6 --warmup 3 --no-getrank --no-cpu-baseline --no-recompute --no-e2e --no-variant > gpurun_out/bench_c4_g$G.json 2> gpurun_out/bench_c4_g$G.err
done
tail -n 3 gpurun_out/grid.log
