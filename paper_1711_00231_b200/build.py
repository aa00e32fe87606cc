"""Build libgraphlb_b200.so in-tree with nvcc for sm_100a.

The shared library is the product: hand-written CUDA kernels + the C-ABI of
include/graphlb_b200.h.  cudart is linked statically so the .so only needs the
driver on the GPU box.
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
BUILD = HERE / "_build"
LIB = HERE / "libgraphlb_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills", "-diag-suppress", "20054"]
SOURCES = ["glb_memory.cu", "glb_graph.cu", "glb_driver.cu", "glb_gen.cu", "glb_peak.cu"]
CXX_SOURCES = ["glb_host_simd.cpp", "glb_io.cpp"]
CXX = os.environ.get("CXX", "g++")
EXTRA = os.environ.get("GLB_EXTRA_FLAGS", "").split()


def _digest() -> str:
    h = hashlib.sha256()
    for p in sorted(CSRC.glob("*")) + [HERE.parent / "include" / "graphlb_b200.h"]:
        h.update(p.name.encode())
        h.update(p.read_bytes())
    h.update(" ".join(ARCH + FLAGS + EXTRA).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    stamp = BUILD / "digest"
    dig = _digest()
    if LIB.exists() and stamp.exists() and stamp.read_text() == dig and not force:
        return LIB
    objs = []
    for src in SOURCES:
        obj = BUILD / (Path(src).stem + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *EXTRA, "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        objs.append(str(obj))
    for src in CXX_SOURCES:  # host-only C++ (AVX2 upload loops)
        obj = BUILD / (Path(src).stem + ".o")
        cmd = [CXX, "-O3", "-mavx2", "-fPIC", "-std=c++17", "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "--cudart", "static", "-o", str(tmp), *objs, "-lpthread"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    stamp.write_text(dig)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
