"""Shared helpers for the GPU parity tests (device buffers via torch, calls via the C-ABI)."""
import numpy as np

from oracle import sambaten as O


def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "the -m gpu tests need a CUDA device (no CPU fallback)"
    return torch


def dev(a, dtype=None):
    """numpy -> contiguous cuda tensor (same bits)."""
    torch = torch_cuda()
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def host(t):
    torch_cuda().cuda.synchronize()
    return t.detach().cpu().numpy()


def rel_fro(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def random_dense(K, J, I, seed, zero_frac=0.0, scale=1.0):
    rng = np.random.default_rng(seed)
    T = (scale * rng.standard_normal((K, J, I))).astype(np.float32)
    if zero_frac:
        T[rng.random(T.shape) < zero_frac] = 0.0
    return T


def oracle_state_from(T0, lam, A, B, C, cfg, cap_entries):
    return O.init_factors(T0, cfg, lam, A, B, C, cap_entries)
