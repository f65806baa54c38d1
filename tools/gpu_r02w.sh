#!/bin/bash
for d in 0 1 2; do PROBE_TAG="dbg$d" SBT_MARG_DBG=$d python tools/marg_probe2.py; done
PROBE_TAG="st72x3" SBT_MARG_STAGE_KB=72 SBT_MARG_RING_KB=216 python tools/marg_probe2.py
PROBE_TAG="dbg2_st72x3" SBT_MARG_DBG=2 SBT_MARG_STAGE_KB=72 SBT_MARG_RING_KB=216 python tools/marg_probe2.py
PROBE_TAG="dbg1_st72x3" SBT_MARG_DBG=1 SBT_MARG_STAGE_KB=72 SBT_MARG_RING_KB=216 python tools/marg_probe2.py
