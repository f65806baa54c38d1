#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_coo.py tests/test_gpu_primitives.py -q -p no:cacheprovider > gpurun_out/coo.log 2>&1; echo "rc=$?" >> gpurun_out/coo.log
timeout 1500 python bench.py --config C5 --steps 4 --warmup 2 --no-getrank --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "rc=$?" >> gpurun_out/bench_c5.err
timeout 900 python bench.py --steps 6 --warmup 3 --no-getrank --no-cpu-baseline --no-e2e --no-variant --no-recompute > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "rc=$?" >> gpurun_out/bench_c4.err
tail -n 3 gpurun_out/coo.log
