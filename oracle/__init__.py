"""Plain, slow, FP64 CPU oracle for SamBaTen's per-batch incremental CP update.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import or run
anything under ``oracle/``.  The product path (``paper_1709_00668_b200``) never
imports it and has no CPU fallback.

The oracle shares no code with the CUDA path (no kernels, headers, helpers,
constants or table generators).  Each function cites the PAPER.md passage
(``P:<line>``) it follows, and, where the paper is silent or garbled, the
reading recorded in DESIGN.md ("Readings", R-numbers = SURVEY.md §8(c) A-numbers).

Parity status per function (pins live in ``tests/test_oracle_*.py``):
  philox4x32_10, uniform53, detlog ........ pinned (Random123 KAT, math.log ulp bound)
  marginals ............................... pinned (brute force, closed form, ||X||_1)
  sample_mode ............................. pinned (exact successive-sampling inclusion
                                            probabilities, s=1, single positive weight)
  gather_dense / gather_coo ............... pinned (coordinate lookup, identity, planted)
  mttkrp .................................. pinned (explicit unfolding x Khatri-Rao,
                                            CP closed form, all-ones example)
  cp_als .................................. pinned (planted noiseless recovery, rank-1,
                                            monotone objective, normalisation invariance)
  match ................................... pinned (identity, known permutation + signs,
                                            brute-force assignment)
  update (merge) .......................... pinned (planted noiseless from truth: C_new
                                            = C_true rows, lambda unchanged, zero-entry cells)
  relative_error / fms .................... pinned (dense materialisation, self-score 1)
"""
from .philox import philox4x32_10, uniform53, detlog  # noqa: F401
from . import sambaten  # noqa: F401
