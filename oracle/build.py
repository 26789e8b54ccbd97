"""Build the CPU oracle (test infrastructure only): oracle/liboracle_pvo.so.

Compiled like the reference's CMake Release build (``-O3 -DNDEBUG``, no
``-march``; proj/CMakeLists.txt:8-10,31) so its timing is a fair stand-in for
the reference CPU path.  The reference itself is unbuildable here (Eigen3,
libpng and the vendored doctest/CLI11/json are absent), so there is no
oracle/_ref build; see DESIGN.md.
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
