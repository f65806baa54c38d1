"""ctypes binding of libsambaten.so (include/sambaten.h).  Argument marshalling only: every
step of the update runs in the library's CUDA kernels.  There is no CPU fallback; if the
library (or a CUDA device) is missing, calls raise."""
import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsambaten.so")

DENSE, COO = 0, 1
MOI_ABS, MOI_SQ = 0, 1

STATUS = {
    0: "OK", -1: "E_INVALID", -2: "E_SHAPE", -3: "E_DEGENERATE", -4: "E_EMPTY_BATCH",
    -5: "E_INDEX_RANGE", -6: "E_NUMERICAL", -7: "E_BATCH_REJECTED", -8: "E_FIXEDPOINT_RANGE",
    -9: "E_OOM", -10: "E_CUDA",
}


class SambatenError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.name = STATUS.get(code, str(code))


class Tensor(C.Structure):
    _fields_ = [("fmt", C.c_int), ("dims", C.c_int64 * 3), ("vals", C.c_void_p),
                ("idx", C.c_void_p * 3), ("nnz", C.c_int64), ("on_device", C.c_int)]


class Opts(C.Structure):
    _fields_ = [("als_max_iters", C.c_int), ("als_tol", C.c_double), ("moi", C.c_int),
                ("s_mode", C.c_int * 3), ("merge_policy", C.c_int), ("accept_tau", C.c_double),
                ("full_fit", C.c_int), ("capacity", C.c_int64), ("capacity_k", C.c_int64),
                ("init_max_iters", C.c_int),
                ("init_tol", C.c_double), ("stream", C.c_void_p), ("borrow_store", C.c_int),
                ("incremental_marginals", C.c_int), ("getrank", C.c_int),
                ("getrank_trials", C.c_int), ("getrank_threshold", C.c_double), ("warm_start", C.c_int),
                ("pipelined", C.c_int)]


class Dist(C.Structure):
    _fields_ = [("rank", C.c_int), ("world", C.c_int), ("nccl_id", C.c_ubyte * 128),
                ("k0", C.c_int64), ("K0_global", C.c_int64)]


class Info(C.Structure):
    _fields_ = [("fit_summary", C.c_double), ("fit_full", C.c_double),
                ("als_iters_max", C.c_int), ("k_total", C.c_int64),
                ("reps_rejected_mask", C.c_uint32), ("scale_exp", C.c_int),
                ("kernel_launches", C.c_int), ("reps_pinv_mask", C.c_uint32),
                ("step_ms", C.c_double * 8), ("als_iters_sum", C.c_int),
                ("rep_rank", C.c_int * 32), ("als_plan", C.c_int * 4),
                ("summary_entries", C.c_int64), ("fit_full_prev", C.c_double),
                ("fit_path", C.c_int)]

    def as_dict(self):
        return dict(fit_summary=self.fit_summary, fit_full=self.fit_full,
                    als_iters_max=self.als_iters_max, k_total=self.k_total,
                    reps_rejected_mask=self.reps_rejected_mask, scale_exp=self.scale_exp,
                    kernel_launches=self.kernel_launches, reps_pinv_mask=self.reps_pinv_mask,
                    step_ms=list(self.step_ms), als_iters_sum=self.als_iters_sum,
                    rep_rank=list(self.rep_rank), als_plan=list(self.als_plan),
                    summary_entries=self.summary_entries, fit_full_prev=self.fit_full_prev,
                    fit_path=self.fit_path)


_lib = None


def lib():
    """Load libsambaten.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1709_00668_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i64, i32, u32, u64, d, ip = C.c_void_p, C.c_int64, C.c_int, C.c_uint32, C.c_uint64, C.c_double, C.c_int
    T, O, I = C.POINTER(Tensor), C.POINTER(Opts), C.POINTER(Info)
    sig = {
        "sambaten_default_opts": (None, [O]),
        "sambaten_init": (i32, [C.POINTER(vp), T, ip, ip, ip, u64, O]),
        "sambaten_init_factors": (i32, [C.POINTER(vp), T, ip, ip, ip, u64, vp, vp, vp, vp, O]),
        "sambaten_update": (i32, [vp, T, vp, vp, vp, vp, I]),
        "sambaten_get_factors": (i32, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                       C.POINTER(i64), C.POINTER(ip)]),
        "sambaten_last_samples": (i32, [vp, vp, vp, vp, C.POINTER(i64)]),
        "sambaten_copy_factors": (i32, [vp, vp, vp, vp, vp]),
        "sambaten_relative_error": (i32, [vp, C.POINTER(d)]),
        "sambaten_checkpoint": (i32, [vp]),
        "sambaten_restore": (i32, [vp]),
        "sambaten_destroy": (None, [vp]),
        "sambaten_fixed_point_scale": (ip, [i64, d]),
        "sambaten_marginals": (i32, [T, ip, ip, vp, vp, vp, vp]),
        "sambaten_sample": (i32, [vp, i64, i64, u64, u32, u32, u32, vp, vp]),
        "sambaten_gather": (i32, [T, vp, i64, vp, i64, vp, i64, vp, vp, vp, vp, vp, i64, vp, vp]),
        "sambaten_mttkrp": (i32, [T, vp, vp, vp, ip, ip, vp, vp]),
        "sambaten_cp_als": (i32, [T, ip, vp, vp, vp, vp, ip, d, vp, vp, vp]),
        "sambaten_fit": (i32, [T, vp, vp, vp, vp, ip, vp, vp]),
        "sambaten_philox": (i32, [u32, u32, u32, u32, u64, i64, vp, vp]),
        "sambaten_detlog": (i32, [vp, i64, vp, vp]),
        "sambaten_dist_unique_id": (i32, [vp]),
        "sambaten_init_factors_dist": (i32, [C.POINTER(vp), T, C.POINTER(Dist), ip, ip, ip, u64, vp, vp, vp, vp, O]),
        "sambaten_batch_partition": (i32, [vp, i64, C.POINTER(i64), C.POINTER(i64)]),
        "sambaten_dist_plan": (i32, [vp, ip, i64, vp, i64, i64, ip, ip, vp, vp]),
        "sambaten_corcondia": (i32, [T, ip, vp, vp, vp, vp, vp, vp]),
        "sambaten_getrank": (i32, [T, ip, ip, u64, ip, d, d, C.POINTER(ip), vp, vp]),
        "sambaten_als_plan": (i32, [ip, ip, ip, ip, ip, vp]),
        "sambaten_recompute": (i32, [vp, ip, d, vp, vp, vp, vp, C.POINTER(d), C.POINTER(ip)]),
        "sambaten_relative_fitness": (i32, [vp, ip, d, C.POINTER(d), C.POINTER(d), C.POINTER(d)]),
        "sambaten_init_dist": (i32, [C.POINTER(vp), T, C.POINTER(Dist), ip, ip, ip, u64, O]),
        "sambaten_last_error": (C.c_char_p, []),
        "sambaten_version": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


EXPORTED = ["sambaten_default_opts", "sambaten_init", "sambaten_init_factors", "sambaten_update",
            "sambaten_get_factors", "sambaten_copy_factors", "sambaten_last_samples", "sambaten_relative_error",
            "sambaten_checkpoint", "sambaten_restore", "sambaten_destroy",
            "sambaten_fixed_point_scale", "sambaten_marginals", "sambaten_sample", "sambaten_gather",
            "sambaten_mttkrp", "sambaten_cp_als", "sambaten_fit", "sambaten_philox", "sambaten_detlog",
            "sambaten_dist_unique_id", "sambaten_init_factors_dist", "sambaten_batch_partition",
            "sambaten_dist_plan", "sambaten_corcondia", "sambaten_getrank", "sambaten_als_plan",
            "sambaten_recompute", "sambaten_relative_fitness", "sambaten_init_dist",
            "sambaten_last_error", "sambaten_version"]


def check(code):
    if code != 0:
        raise SambatenError(code, lib().sambaten_last_error().decode())


# ----------------------------------------------------------------------------------------
# marshalling helpers (torch tensors on cuda/cpu, or numpy arrays)
# ----------------------------------------------------------------------------------------
def ptr(x):
    """Raw data pointer of a torch tensor or numpy array (None -> NULL)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor passed to the C-ABI must be contiguous")
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array passed to the C-ABI must be C-contiguous (row-major)")
        return x.ctypes.data
    if isinstance(x, int):
        return x
    raise TypeError(type(x))


def _on_device(x):
    return int(bool(getattr(x, "is_cuda", False)))


def dense(T):
    """sambaten_tensor for a contiguous float32 array of shape (K, J, I) (i fastest)."""
    K, J, I = T.shape
    t = Tensor()
    t.fmt = DENSE
    t.dims[0], t.dims[1], t.dims[2] = I, J, K
    t.vals = ptr(T)
    t.nnz = 0
    t.on_device = _on_device(T)
    t._keep = (T,)
    return t


def coo(i, j, k, v, dims):
    t = Tensor()
    t.fmt = COO
    t.dims[0], t.dims[1], t.dims[2] = dims
    t.vals = ptr(v)
    t.idx[0], t.idx[1], t.idx[2] = ptr(i), ptr(j), ptr(k)
    t.nnz = int(v.shape[0])
    t.on_device = _on_device(v)
    t._keep = (i, j, k, v)
    return t


def default_opts(**kw):
    o = Opts()
    lib().sambaten_default_opts(C.byref(o))
    for key, val in kw.items():
        if key == "s_mode":
            for m in range(3):
                o.s_mode[m] = int(val[m])
        elif key == "stream":
            o.stream = val
        else:
            setattr(o, key, val)
    return o


def stream_ptr(stream):
    """cudaStream_t of a torch.cuda.Stream (or None for the legacy default stream)."""
    if stream is None:
        return None
    return stream.cuda_stream


# ----------------------------------------------------------------------------------------
# handle API with the C names
# ----------------------------------------------------------------------------------------
def sambaten_init(X0, R, s, r, seed, opts=None):
    h = C.c_void_p()
    check(lib().sambaten_init(C.byref(h), C.byref(X0), R, s, r, seed, C.byref(opts) if opts else None))
    return h


def _c_in(x):
    """Input-only host array: row-major copy if needed (factors are [rows][R] row-major)."""
    return np.ascontiguousarray(x) if isinstance(x, np.ndarray) else x


def sambaten_init_factors(X0, R, s, r, seed, A, B, Cm, lam, opts=None):
    A, B, Cm, lam = _c_in(A), _c_in(B), _c_in(Cm), _c_in(lam)
    h = C.c_void_p()
    check(lib().sambaten_init_factors(C.byref(h), C.byref(X0), R, s, r, seed, ptr(A), ptr(B), ptr(Cm),
                                      ptr(lam), C.byref(opts) if opts else None))
    return h


def sambaten_dist_unique_id():
    buf = (C.c_ubyte * 128)()
    check(lib().sambaten_dist_unique_id(buf))
    return bytes(buf)


def make_dist(rank, world, nccl_id, k0, K0_global):
    d = Dist()
    d.rank, d.world, d.k0, d.K0_global = rank, world, k0, K0_global
    C.memmove(d.nccl_id, nccl_id, 128)
    return d


def sambaten_init_factors_dist(X0_local, dist, R, s, r, seed, A, B, Cm, lam, opts=None):
    A, B, Cm, lam = _c_in(A), _c_in(B), _c_in(Cm), _c_in(lam)
    h = C.c_void_p()
    check(lib().sambaten_init_factors_dist(C.byref(h), C.byref(X0_local), C.byref(dist), R, s, r, seed, ptr(A),
                                           ptr(B), ptr(Cm), ptr(lam), C.byref(opts) if opts else None))
    return h


def sambaten_dist_plan(Kp, owner_old, K_old, K_new, world, rank):
    """Host-only exchange plan (no GPU): (send_slices[world], recv_slices[world])."""
    Kp = np.ascontiguousarray(Kp, np.int32)
    owner_old = np.ascontiguousarray(owner_old, np.int32)
    send = np.zeros(world, np.int64)
    recv = np.zeros(world, np.int64)
    check(lib().sambaten_dist_plan(ptr(Kp), Kp.shape[0], Kp.shape[1], ptr(owner_old), K_old, K_new, world,
                                   rank, ptr(send), ptr(recv)))
    return send, recv


def sambaten_batch_partition(h, K_new):
    b, n = C.c_int64(), C.c_int64()
    check(lib().sambaten_batch_partition(h, K_new, C.byref(b), C.byref(n)))
    return b.value, n.value


def sambaten_update(h, batch, A=None, B=None, Cm=None, lam=None):
    info = Info()
    check(lib().sambaten_update(h, C.byref(batch), ptr(A), ptr(B), ptr(Cm), ptr(lam), C.byref(info)))
    return info


def sambaten_get_factors(h):
    a, b, c, l = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
    dims = (C.c_int64 * 3)()
    R = C.c_int()
    check(lib().sambaten_get_factors(h, C.byref(a), C.byref(b), C.byref(c), C.byref(l), dims, C.byref(R)))
    return dict(A=a.value, B=b.value, C=c.value, lam=l.value, dims=tuple(dims), R=R.value)


def sambaten_copy_factors(h, A=None, B=None, Cm=None, lam=None):
    check(lib().sambaten_copy_factors(h, ptr(A), ptr(B), ptr(Cm), ptr(lam)))


def sambaten_last_samples(h, Is=None, Js=None, Ks=None):
    n = (C.c_int64 * 3)()
    check(lib().sambaten_last_samples(h, ptr(Is), ptr(Js), ptr(Ks), n))
    return tuple(n)


def sambaten_recompute(h, max_iters, tol, A=None, B=None, Cm=None, lam=None):
    """CP_ALS baseline: full CP-ALS of the handle's current tensor; returns
    (relative error, iterations); factors copied into the given arrays when not None."""
    e, it = C.c_double(), C.c_int()
    check(lib().sambaten_recompute(h, max_iters, tol, ptr(A), ptr(B), ptr(Cm), ptr(lam), C.byref(e), C.byref(it)))
    return e.value, it.value


def sambaten_relative_fitness(h, max_iters, tol):
    """Relative fitness: (rf, relerr_sambaten, relerr_cp_als)."""
    rf, es, eb = C.c_double(), C.c_double(), C.c_double()
    check(lib().sambaten_relative_fitness(h, max_iters, tol, C.byref(rf), C.byref(es), C.byref(eb)))
    return rf.value, es.value, eb.value


def sambaten_init_dist(X0_local, dist, R, s, r, seed, opts=None):
    h = C.c_void_p()
    check(lib().sambaten_init_dist(C.byref(h), C.byref(X0_local), C.byref(dist), R, s, r, seed,
                                   C.byref(opts) if opts else None))
    return h


def sambaten_relative_error(h):
    v = C.c_double()
    check(lib().sambaten_relative_error(h, C.byref(v)))
    return v.value


def sambaten_checkpoint(h):
    check(lib().sambaten_checkpoint(h))


def sambaten_restore(h):
    check(lib().sambaten_restore(h))


def sambaten_destroy(h):
    lib().sambaten_destroy(h)


def sambaten_fixed_point_scale(cap, max_phi):
    return lib().sambaten_fixed_point_scale(int(cap), float(max_phi))


def sambaten_marginals(X, moi, S, x1, x2, x3, stream=None):
    check(lib().sambaten_marginals(C.byref(X), moi, S, ptr(x1), ptr(x2), ptr(x3), stream))


def sambaten_sample(w, n, n_s, seed, update_id, rep, mode, out, stream=None):
    check(lib().sambaten_sample(ptr(w), n, n_s, seed, update_id, rep, mode, ptr(out), stream))


def sambaten_gather(X, Is, nI, Js, nJ, Ks, nK, out_dense=None, oi=None, oj=None, ok=None, ov=None,
                    cap=0, out_nnz=None, stream=None):
    check(lib().sambaten_gather(C.byref(X), ptr(Is), nI, ptr(Js), nJ, ptr(Ks), nK, ptr(out_dense),
                                ptr(oi), ptr(oj), ptr(ok), ptr(ov), cap, ptr(out_nnz), stream))


def sambaten_mttkrp(X, U0, U1, U2, R, mode, M, stream=None):
    check(lib().sambaten_mttkrp(C.byref(X), ptr(U0), ptr(U1), ptr(U2), R, mode, ptr(M), stream))


def sambaten_cp_als(X, R, U0, U1, U2, lam_out, max_iters, tol, fit_out, iters_out, stream=None):
    check(lib().sambaten_cp_als(C.byref(X), R, ptr(U0), ptr(U1), ptr(U2), ptr(lam_out), max_iters, tol,
                                ptr(fit_out), ptr(iters_out), stream))


def sambaten_fit(X, lam, A, B, Cm, R, relerr, stream=None):
    check(lib().sambaten_fit(C.byref(X), ptr(lam), ptr(A), ptr(B), ptr(Cm), R, ptr(relerr), stream))


def sambaten_als_plan(nI, nJ, nK, R, r):
    """The a4 plan [kind, CTAs per rep, RB, D in smem] the library picks for r summaries of
    shape nI x nJ x nK at rank R (sambaten_info.als_plan layout)."""
    out = np.zeros(4, np.int32)
    check(lib().sambaten_als_plan(nI, nJ, nK, R, r, out.ctypes.data))
    return [int(x) for x in out]


def sambaten_corcondia(X, F, A, B, Cm, lam, stream=None):
    """CorConDia (R29) of [[lam; A, B, C]] (device fp32 factors, device fp64 lam) of dense X."""
    out = np.zeros(1, np.float64)
    check(lib().sambaten_corcondia(C.byref(X), F, ptr(A), ptr(B), ptr(Cm), ptr(lam), ptr(out), stream))
    return float(out[0])


def sambaten_getrank(X, R_max, trials, seed, max_iters, tol, threshold=90.0, stream=None):
    """GetRank (Alg. 2, R29-R31) of dense X: (R_new, cc[R_max][trials])."""
    cc = np.zeros((R_max, trials), np.float64)
    rn = C.c_int(0)
    check(lib().sambaten_getrank(C.byref(X), R_max, trials, seed, max_iters, tol, threshold, C.byref(rn),
                                 ptr(cc), stream))
    return rn.value, cc


def sambaten_philox(c0, c1, c2, c3, key, n, out, stream=None):
    check(lib().sambaten_philox(c0, c1, c2, c3, key, n, ptr(out), stream))


def sambaten_detlog(u, n, out, stream=None):
    check(lib().sambaten_detlog(ptr(u), n, ptr(out), stream))
