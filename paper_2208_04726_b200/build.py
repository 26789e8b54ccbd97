"""Build the sm_100a shared library ``libpvo_b200.so`` in-tree.

``python paper_2208_04726_b200/build.py`` (or ``__graft_entry__.build()``)
compiles every CUDA/C++ source under ``csrc/`` with nvcc for
``-gencode arch=compute_100a,code=sm_100a`` and links the C-ABI library next
to this file, where the ctypes loader finds it.  nvcc cross-compiles, so this
works on a machine without a GPU.  Objects are cached under ``build/`` and
rebuilt when a source or header is newer.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "pvo_b200"
LIB = PKG / "libpvo_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "--expt-relaxed-constexpr",
    "-Xcompiler",
    "-fPIC",
    "-Xcompiler",
    "-Wall",
    "-I",
    str(ROOT / "include"),
]
SOURCES = ["corr.cu", "corr_tma.cu", "ba.cu", "ba_large.cu", "measure.cu", "dgraph.cu", "features.cu", "capi_core.cu", "capi_window.cu",
           "capi_provider.cu", "capi_batch.cu", "capi_dgraph.cu", "graph.cpp"]
# per-file extra flags: the provider measurement rounds every product / sum like the
# x86-64 reference build (no FMA contraction), so its discrete decisions agree
EXTRA = {"measure.cu": ["--fmad=false"], "features.cu": ["--fmad=false"]}


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found; the sm_100a library cannot be built")
    return cand


def _headers() -> list[Path]:
    return list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + list((ROOT / "include").glob("*.h"))


def build(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    newest_header = max((h.stat().st_mtime for h in _headers()), default=0.0)
    objs = []
    for src in SOURCES:
        s = CSRC / src
        o = BUILD / (src + ".o")
        objs.append(o)
        if not force and o.exists() and o.stat().st_mtime >= max(s.stat().st_mtime, newest_header):
            continue
        cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *EXTRA.get(src, []), "-c", str(s), "-o", str(o)]
        if src.endswith(".cu"):
            cmd[1:1] = ["-Xptxas", "-v"] if verbose else []
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    if force or not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
