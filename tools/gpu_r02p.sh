#!/bin/bash
mkdir -p gpurun_out
P=tools/coo_marg_probe.py
( for nr in 8 16 24; do PROBE_TAG="nrep$nr" SBT_MARG_NREP=$nr python $P; done
for b in 4 16; do PROBE_TAG="bps$b" SBT_MARG_BPS=$b python $P; done ) > gpurun_out/cmp.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_primitives.py -q -p no:cacheprovider -k marginals >> gpurun_out/cmp.txt 2>&1
timeout 600 ncu --set full --import-source on -k regex:marg_coo_rep -c 1 -o gpurun_out/prof_r02_coo_marg2 python $P > gpurun_out/ncu_coo_marg.log 2>&1
cat gpurun_out/cmp.txt | tail -12
