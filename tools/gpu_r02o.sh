#!/bin/bash
mkdir -p gpurun_out
P=tools/coo_marg_probe.py
( PROBE_TAG=norep SAMBATEN_COO_MARG_NOREP=1 python $P
for nr in 4 16 32 64; do PROBE_TAG="nrep$nr" SBT_MARG_NREP=$nr python $P; done
for b in 2 4 16; do PROBE_TAG="bps$b" SBT_MARG_BPS=$b SBT_MARG_NREP=16 python $P; done ) > gpurun_out/cmp.txt 2>&1
SBT_MARG_NREP=16 timeout 600 ncu --set full --import-source on -k regex:marg_coo_rep -c 1 -o gpurun_out/prof_r02_coo_marg python $P > gpurun_out/ncu_coo_marg.log 2>&1
cat gpurun_out/cmp.txt
