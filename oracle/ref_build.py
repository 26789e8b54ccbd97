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
* pvo_dropin_tests - the SAME reference tests linked against the product's
                    drop-in operator layer instead: the reference's sources
                    minus camera.cpp / correlation.cpp / bundle_adjust.cpp,
                    plus paper_2208_04726_b200/dropin/*.cpp (the reference's
                    declared operators implemented over the C-ABI) and
                    libpvo_b200.so.  Run on the GPU box by tests/test_dropin.py:
                    the reference's own test cases exercise the sm_100a
                    kernels through the reference's C++ signatures.

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
DROPIN_TESTS = OUT / "pvo_dropin_tests"
PKG = ROOT / "paper_2208_04726_b200"
DROPIN = PKG / "dropin"
# reference translation units the drop-in layer replaces
DROPIN_REPLACES = {"camera", "correlation", "bundle_adjust"}


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
    build_dropin(objs[: len(LIB_SOURCES)], test_objs, force)
    return LIB


def build_dropin(lib_objs: list[Path], test_objs: list[Path], force: bool = False) -> Path | None:
    """Link the reference's tests against the drop-in layer + libpvo_b200.so."""
    so = PKG / "libpvo_b200.so"
    if not so.exists():
        return None
    extra = ["-I", str(ROOT / "include"), "-I", str(DROPIN)]
    jobs = [(src, OBJ / f"{src.stem}.o", extra) for src in sorted(DROPIN.glob("*.cpp"))]
    deps_newest = max(p.stat().st_mtime for p in DROPIN.glob("*.hpp"))
    for src, obj, ex in jobs:
        if obj.exists() and obj.stat().st_mtime < deps_newest:
            obj.unlink()
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex_:
        drop_objs = list(ex_.map(lambda j: _compile(*j), jobs))
    kept = [o for o in lib_objs if o.stem not in DROPIN_REPLACES]
    newest = max(o.stat().st_mtime for o in drop_objs + kept + test_objs + [so])
    if force or not DROPIN_TESTS.exists() or DROPIN_TESTS.stat().st_mtime < newest:
        tmp = DROPIN_TESTS.with_suffix(".tmp")
        rpath = "-Wl,-rpath,$ORIGIN/../../paper_2208_04726_b200"
        subprocess.run(FLAGS + [*map(str, test_objs), *map(str, kept), *map(str, drop_objs), "-L", str(PKG),
                                "-lpvo_b200", rpath, "-o", str(tmp)], check=True)
        os.replace(tmp, DROPIN_TESTS)
    return DROPIN_TESTS


if __name__ == "__main__":
    print(build(force="-f" in sys.argv))
