"""ctypes binding of synth/libsynthgen.so (synth/csrc/gen.cu): the on-device generator of the
large dense planted configs.  Input tooling only (no SamBaTen arithmetic); built by
synth.gpu.build() (called from __graft_entry__.build())."""
import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "gen.cu")
LIB = os.path.join(HERE, "libsynthgen.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
_lib = None


def build(force=False):
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-shared",
           "-Xcompiler", "-fPIC", "-cudart", "static", "-o", LIB + ".tmp", SRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {SRC}:\n{r.stdout}\n{r.stderr}")
    os.replace(LIB + ".tmp", LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} is not built (synth.gpu.build())")
        _lib = C.CDLL(LIB)
        _lib.synth_dense_slab.restype = C.c_int
        _lib.synth_dense_slab.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                          C.c_int, C.c_int64, C.c_int64, C.c_double, C.c_uint64, C.c_void_p]
    return _lib


def dense_slab(out, A, B, Cm, sigma, seed, k0, nk, stream=0):
    """Fill the contiguous float32 CUDA tensor ``out`` ([nk, J, I]) with slices [k0, k0+nk) of
    the planted tensor; A, B, Cm: contiguous float64 CUDA tensors (Cm holds all K rows)."""
    I, R = A.shape
    J = B.shape[0]
    assert out.is_cuda and out.is_contiguous() and out.numel() == nk * J * I
    for t in (A, B, Cm):
        assert t.is_cuda and t.is_contiguous() and str(t.dtype) == "torch.float64"
    e = lib().synth_dense_slab(out.data_ptr(), A.data_ptr(), B.data_ptr(), Cm.data_ptr(), I, J, R, k0, nk,
                               float(sigma), int(seed), stream)
    if e != 0:
        raise RuntimeError(f"synth_dense_slab failed: cudaError {e}")
