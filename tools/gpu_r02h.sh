#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_update.py -q -p no:cacheprovider -k pipelined > gpurun_out/pipe.log 2>&1; echo "rc=$?" >> gpurun_out/pipe.log
timeout 1500 python bench.py --steps 6 --warmup 3 --no-getrank --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?" >> gpurun_out/bench_c4.err
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/pipe.log gpurun_out/pytest_gpu.log
