"""Build libmfwq.so in-tree with nvcc for sm_100a (no torch extension machinery).

    python -m paper_1712_08565_b200.build [--force]

Objects go to build/, the shared library to paper_1712_08565_b200/libmfwq.so.
"""

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", os.environ.get("MFWQ_BUILD_TAG", "mfwq"))
LIB = os.environ.get("MFWQ_BUILD_LIB") or os.path.join(PKG, "libmfwq.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include():
    """nccl.h of the NCCL torch bundles (types only: libmfwq.so dlopens that library at run time)."""
    try:
        import nvidia.nccl as nc
        base = list(nc.__path__)[0]
    except ImportError:
        base = ""
    inc = os.path.join(base, "include")
    if not os.path.exists(os.path.join(inc, "nccl.h")):
        raise RuntimeError("nccl.h of torch's bundled NCCL (nvidia.nccl) not found")
    return inc


FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", _nccl_include()] + \
    os.environ.get("MFWQ_NVCC_EXTRA", "").split()
SOURCES = ["rule1d.cpp", "stiffness.cu", "fused2.cu", "fused2_otf.cu", "fused3.cu", "fd.cu", "modal_gemm.cu", "pcg.cu",
           "bicgstab.cu", "quadrature.cu", "dist.cu", "capi.cu"]
LIBS = ["-lcusolver", "-ldl", "-Xlinker", "-rpath,/usr/local/cuda/lib64", "-L/usr/local/cuda/lib64"]


def _deps_mtime():
    ts = [os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC)]
    ts.append(os.path.getmtime(os.path.join(ROOT, "include", "mfwq.h")))
    ts.append(os.path.getmtime(__file__))
    return max(ts)


def _compile(src, verbose):
    obj = os.path.join(BUILD, src + ".o")
    cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
    if src.endswith(".cu") and os.environ.get("MFWQ_PTXAS_V"):
        cmd += ["-Xptxas", "-v"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip() and os.environ.get("MFWQ_PTXAS_V"):
        print(r.stderr, file=sys.stderr)
    return obj


def build(force=False, verbose=False):
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _deps_mtime():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, *LIBS]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
