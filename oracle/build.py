"""Build the CPU oracle (test infrastructure only): oracle/liboracle_pvo.so.

Compiled like the reference's CMake Release build (``-O3 -DNDEBUG``, no
``-march``; proj/CMakeLists.txt:8-10,31) so its timing is a fair stand-in for
the reference CPU path.  When /root/reference is present (this container,
not the GPU box), it also builds oracle/_ref from the reference's own sources
(oracle/ref_build.py: the reference compiled unmodified against in-repo shims
for the absent Eigen3 / doctest / json / libpng).
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
SRC = HERE / "pvo_oracle.cpp"
LIB = HERE / "liboracle_pvo.so"


def build(force: bool = False) -> Path:
    import importlib.util

    spec = importlib.util.spec_from_file_location("oracle_ref_build", HERE / "ref_build.py")
    ref_build = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ref_build)
    ref_build.build(force=force)
    return _build_restated(force)


def _build_restated(force: bool) -> Path:
    if not force and LIB.exists() and LIB.stat().st_mtime >= SRC.stat().st_mtime:
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    cmd = ["g++", "-std=c++20", "-O3", "-DNDEBUG", "-Wall", "-Wextra", "-shared", "-fPIC", "-pthread",
           str(SRC), "-o", str(tmp)]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="-f" in sys.argv))
