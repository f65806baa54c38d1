"""Seeded synthetic inputs shared by tests/ and bench.py.

This module holds NONE of SamBaTen's arithmetic (no marginals, sampling, gather, ALS,
matching or merge): it only builds planted tensors and the BASELINE.json configs, so
both the oracle and the CUDA path can be fed the very same bits.  Recipes are
described in DESIGN.md ("Synthetic inputs"); they stand in for the paper's synthetic
generator (Table 2) and for the FROSTT datasets (Table 3
P:378-405), which are not available.
"""
from .planted import (planted_dense, planted_dense_factors, dense_from_factors,  # noqa: F401
                      community_coo, zipf_planted_coo, split_dense, split_coo, CooArrays)
from .configs import CONFIGS, Workload  # noqa: F401
