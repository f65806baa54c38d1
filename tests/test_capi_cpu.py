"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/sambaten.h
declares, and its host-only helpers agree with the oracle (no GPU compute calls)."""
import os
import re

from oracle import sambaten as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "sambaten.h")).read()
    return sorted(set(re.findall(r"SAMBATEN_API\s+[\w\s\*]*?\b(sambaten_\w+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_1709_00668_b200 import _lib
    L = _lib.lib()
    syms = _header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTED)


def test_version_and_default_opts():
    from paper_1709_00668_b200 import _lib
    assert b"sm_100a" in _lib.lib().sambaten_version()
    o = _lib.default_opts()
    assert o.als_max_iters == 30 and o.accept_tau == 0.9 and o.init_max_iters == 1000
    assert o.moi == 0 and o.merge_policy == 0
    # the fields appended last are filled by the C side: a ctypes layout that drifted from the
    # header would read them at the wrong offsets
    assert o.getrank == 0 and o.getrank_trials == 1 and o.getrank_threshold == 90.0
    assert o.warm_start == 0 and o.incremental_marginals == 0 and o.borrow_store == 0


def test_fixed_point_scale_matches_oracle():
    from paper_1709_00668_b200 import _lib
    for cap, mx in ((125_000, 3.0), (3000 ** 3, 10.0), (2_100_000, 65.0), (105_000_000, 1.5),
                    (1, 1.0), (10, 2.0 ** -40), (2 ** 40, 2.0 ** 50), (12345, 0.75)):
        assert _lib.sambaten_fixed_point_scale(cap, mx) == O.fixed_point_scale(cap, mx)


def test_no_gpu_means_loud_failure():
    """Without a CUDA device a compute call must fail (no CPU fallback)."""
    import numpy as np
    import torch
    from paper_1709_00668_b200 import _lib
    if torch.cuda.is_available():
        return
    T = np.ones((2, 2, 2), np.float32)
    try:
        _lib.sambaten_init_factors(_lib.dense(T), 1, 1, 1, 0, np.ones((2, 1), np.float32),
                                   np.ones((2, 1), np.float32), np.ones((2, 1), np.float32),
                                   np.ones(1, np.float32))
    except _lib.SambatenError as e:
        assert e.name in ("E_CUDA",)
    else:
        raise AssertionError("init succeeded without a GPU")
from paper_1709_00668_b200 import _lib as L
def test_ptr_rejects_non_row_major():
    import numpy as np
    import pytest
    from paper_1709_00668_b200 import _lib as L
    a = np.asfortranarray(np.ones((5, 3), np.float32))
    with pytest.raises(ValueError):
        L.ptr(a)
    assert L.ptr(np.ascontiguousarray(a)) is not None
