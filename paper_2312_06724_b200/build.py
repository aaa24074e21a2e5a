"""Build libbhpp.so (the CUDA engine + C ABI) in-tree for sm_100a.

    python -m paper_2312_06724_b200.build [--force]

Output: paper_2312_06724_b200/_lib/libbhpp.so (git-ignored; it travels to the
GPU box with the gpurun snapshot).  nvcc cross-compiles here without a GPU.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "_lib"
LIB = LIB_DIR / "libbhpp.so"
INCLUDE = PKG.parent / "include"
SOURCES = ["engine.cu", "graph_store.cu", "csr_build.cu", "edge_list.cpp", "walks.cu", "alias.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.cpp")) + list(INCLUDE.glob("*.h")) + [Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps)


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    LIB_DIR.mkdir(exist_ok=True)
    obj_dir = LIB_DIR / "obj"
    obj_dir.mkdir(exist_ok=True)
    tmp = LIB.with_suffix(".so.tmp")
    flags = [
        *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
        "-Xcompiler", "-O2", "--expt-relaxed-constexpr", "-I", str(INCLUDE),
        *(["-Xptxas", "-v"] if verbose else []),
    ]
    # one nvcc per translation unit, in parallel, then one link
    procs, objs = [], []
    for src in SOURCES:
        obj = obj_dir / (src + ".o")
        objs.append(obj)
        procs.append((src, subprocess.Popen([nvcc(), *flags, "-c", "-o", str(obj), str(CSRC / src)])))
    failed = [src for src, p in procs if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, f"nvcc {' '.join(failed)}")
    subprocess.run([nvcc(), *ARCH, "-shared", "-o", str(tmp), *[str(o) for o in objs]], check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
