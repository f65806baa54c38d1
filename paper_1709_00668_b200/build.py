"""Build libsambaten.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_1709_00668_b200.build [--force]

Objects go to paper_1709_00668_b200/build/; the shared library to
paper_1709_00668_b200/libsambaten.so (git-ignored, travels to the GPU box with gpurun).
"""
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libsambaten.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NCCL_DIR = os.environ.get("SBT_NCCL_DIR", "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr", "-cudart", "static",
    "-I", os.path.join(ROOT, "include"),
    "-I", os.path.join(NCCL_DIR, "include"),
]


def _deps_mtime():
    files = glob.glob(os.path.join(CSRC, "*")) + [os.path.join(ROOT, "include", "sambaten.h")]  # incl. *.inc
    return max(os.path.getmtime(f) for f in files)


def _compile(src):
    obj = os.path.join(OUT_DIR, os.path.basename(src) + ".o")
    cmd = [NVCC, *FLAGS, "-c", src, "-o", obj]
    if os.environ.get("SBT_EXTRA_FLAGS"):
        cmd += os.environ["SBT_EXTRA_FLAGS"].split()
    if os.environ.get("SBT_PTXAS_V"):
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force=False, verbose=False):
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _deps_mtime():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        results = list(ex.map(_compile, srcs))
    if verbose:
        for _, err in results:
            if err.strip():
                print(err)
    objs = [o for o, _ in results]
    tmp = LIB + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o", tmp, *objs,
           "-L", os.path.join(NCCL_DIR, "lib"), "-l:libnccl.so.2",
           "-Xlinker", "-rpath=" + os.path.join(NCCL_DIR, "lib")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
