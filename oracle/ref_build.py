"""Build oracle/_ref from the reference's own sources (test infrastructure only).

Compiles /root/reference/proj/src/*.cpp UNMODIFIED, in place (nothing is
copied into the repo), against the in-repo shims for the libraries this image
lacks (oracle/ref_shim/: an Eigen 3 subset, doctest, nlohmann::json, a libpng
stub), with the reference's Release flags (-O3 -DNDEBUG, no -march;
proj/CMakeLists.txt:8-10,31).  Outputs, all under oracle/_ref/ (git-ignored,
travels to the GPU box with the snapshot):

* libpvo_ref.so   - the reference library + oracle/ref_capi.cpp, exporting the
                    same orc_* surface as the restatement (oracle/pyoracle.py
                    prefers it when present);
* pvo_ref_tests   - the reference's own unit tests (proj/tests/test_*.cpp,
                    doctest suites se3 camera patch_graph bundle_adjust
                    features simulator trajectory pipeline) linked against it.

The reference's CMake build itself is not run (it needs cmake + system
Eigen/libpng/vendor trees); this script is the committed recipe instead.
Usage: python oracle/ref_build.py [-f]
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
REF = Path(os.environ.get("PVO_REFERENCE", "/root/reference")) / "proj"
OUT = HERE / "_ref"
OBJ = ROOT / "build" / "ref"
SHIM = HERE / "ref_shim"

LIB_SOURCES = ["se3", "camera", "image", "patch_graph", "bundle_adjust", "features", "correlation",
               "flow_provider", "simulator", "trajectory", "pipeline", "runner"]
TEST_SOURCES = ["test_main", "test_se3", "test_camera", "test_patch_graph", "test_bundle_adjust", "test_features",
                "test_simulator", "test_trajectory", "test_pipeline"]
FLAGS = ["g++", "-std=c++20", "-O3", "-DNDEBUG", "-fPIC", "-pthread", "-w", "-I", str(SHIM), "-I",
         str(REF / "include")]

LIB = OUT / "libpvo_ref.so"
TESTS = OUT / "pvo_ref_tests"


def available() -> bool:
    return (REF / "src" / "bundle_adjust.cpp").exists()


def _compile(src: Path, obj: Path, extra: list[str]) -> Path:
    deps = [src] + list(SHIM.rglob("*")) + list((REF / "include" / "pvo").glob("*.hpp"))
    if obj.exists() and obj.stat().st_mtime >= max(d.stat().st_mtime for d in deps if d.is_file()):
        return obj
    obj.parent.mkdir(parents=True, exist_ok=True)
    tmp = obj.with_suffix(".o.tmp")
    subprocess.run(FLAGS + extra + ["-c", str(src), "-o", str(tmp)], check=True)
    os.replace(tmp, obj)
    return obj


def build(force: bool = False) -> Path | None:
    if not available():
        return LIB if LIB.exists() else None  # GPU box: use the prebuilt library that travelled
    OUT.mkdir(parents=True, exist_ok=True)
    if force:
        for o in OBJ.glob("*.o"):
            o.unlink()
    jobs = [(REF / "src" / f"{s}.cpp", OBJ / f"{s}.o", []) for s in LIB_SOURCES]
    jobs.append((HERE / "ref_capi.cpp", OBJ / "ref_capi.o", []))
    jobs += [(REF / "tests" / f"{s}.cpp", OBJ / f"{s}.o", ["-I", str(REF / "tests")]) for s in TEST_SOURCES]
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda j: _compile(*j), jobs))
    lib_objs = objs[: len(LIB_SOURCES)]
    capi_obj = objs[len(LIB_SOURCES)]
    test_objs = objs[len(LIB_SOURCES) + 1:]
    newest = max(o.stat().st_mtime for o in objs)
    if force or not LIB.exists() or LIB.stat().st_mtime < newest:
        tmp = LIB.with_suffix(".so.tmp")
        subprocess.run(FLAGS + ["-shared", *map(str, lib_objs), str(capi_obj), "-o", str(tmp)], check=True)
        os.replace(tmp, LIB)
    if force or not TESTS.exists() or TESTS.stat().st_mtime < newest:
        tmp = TESTS.with_suffix(".tmp")
        subprocess.run(FLAGS + [*map(str, test_objs), *map(str, lib_objs), "-o", str(tmp)], check=True)
        os.replace(tmp, TESTS)
    return LIB


if __name__ == "__main__":
    print(build(force="-f" in sys.argv))
