#!/bin/bash
# round-2 check: new edge-case parity tests, the full GPU suite, the C4 default bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_edges.py -q -p no:cacheprovider -rA --durations=10 > gpurun_out/edges.log 2>&1; echo "edges rc=$?" >> gpurun_out/edges.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_edges.py::test_c4_summary_shape_parity > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
SAMBATEN_DEBUG=0 timeout 1500 python bench.py --steps 4 --warmup 3 --no-getrank > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?" >> gpurun_out/bench_c4.err
tail -5 gpurun_out/edges.log; tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench_c4.err; head -c 3000 gpurun_out/bench_c4.json
