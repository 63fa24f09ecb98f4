"""Build the C-ABI shared library libmxq200.so for sm_100a (in-tree).

nvcc -gencode arch=compute_100a,code=sm_100a (NOT -arch=sm_100a, which also
embeds compute_100 PTX and rejects tcgen05), -lineinfo for ncu source
correlation, no fast-math / FTZ (the quantizer arithmetic is bit-exact and
f32 subnormals matter).  The CUDA runtime is linked
statically so the library has no dependency on a particular libcudart.
"""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libmxq200.so")
SOURCES = ["capi.cu", "quantize.cu", "qsnr.cu", "layout.cu", "gemm_exact.cu", "gemm_tc.cu", "gemm_mbs.cu"]
HEADERS = ["sq_dev.cuh", "mxq_arith.cuh", "mxq_device.cuh", "mxq_internal.h", "tc_ptx.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "-ftz=false", "-prec-div=true", "-prec-sqrt=true", "-fmad=true",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-v",
]
# Development builds only (e.g. MXQ_NVCC_EXTRA=-DMXQ_GEMM_TRACE=1 for tools/trace_mbs.py).
FLAGS += os.environ.get("MXQ_NVCC_EXTRA", "").split()


def _digest() -> str:
    h = hashlib.sha256()
    for f in SOURCES + HEADERS:
        p = os.path.join(CSRC, f)
        if os.path.exists(p):
            h.update(open(p, "rb").read())
    h.update(open(os.path.join(HERE, "..", "include", "mxq200.h"), "rb").read())
    h.update(" ".join(FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    stamp = os.path.join(OUT_DIR, "libmxq200.sha256")
    digest = _digest()
    if not force and os.path.exists(LIB) and os.path.exists(stamp) and open(stamp).read().strip() == digest:
        return LIB
    objs = []
    for src in SOURCES:
        obj = os.path.join(OUT_DIR, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError(f"nvcc failed on {src}")
        objs.append(obj)
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB, *objs, "-cudart", "static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    with open(stamp, "w") as fh:
        fh.write(digest)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
