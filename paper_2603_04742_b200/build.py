"""In-tree build of the native library ``lib/libcssc_he.so``.

Compiles every CUDA source for sm_100a (``-gencode arch=compute_100a,code=sm_100a
-lineinfo``) and the host C++ with g++ (C++20), then links one shared
library that exports the C-ABI declared in ``include/spmvgpu.h``.  Objects go
to ``build/`` next to this file; rebuilds are incremental on source/header
mtimes.  Also builds the test-side checkers under ``oracle/`` when asked
(they are never linked into the product).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
# CSSC_BUILD_TAG / CSSC_NVCC_DEFINES: a variant build (A/B experiments) into
# build_<tag>/ and lib/libcssc_he_<tag>.so, loaded with CSSC_LIB
_TAG = os.environ.get("CSSC_BUILD_TAG", "")
_DEFS = os.environ.get("CSSC_NVCC_DEFINES", "").split()
BUILD = PKG / ("build_" + _TAG if _TAG else "build")
LIBDIR = PKG / "lib"
LIB = LIBDIR / ("libcssc_he_" + _TAG + ".so" if _TAG else "libcssc_he.so")
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INCLUDES = [f"-I{ROOT / 'include'}", f"-I{CSRC}", f"-I{CUDA_HOME / 'include'}"]


def _sources():
    cu = sorted(CSRC.glob("*.cu"))
    cpp = sorted(CSRC.glob("*.cpp")) + sorted((CSRC / "host").glob("*.cpp"))
    return cu, cpp


def _headers():
    hs = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + list((CSRC / "host").glob("*.hpp"))
    hs += list((ROOT / "include").rglob("*.h*"))
    return hs


def _obj(src: Path) -> Path:
    rel = src.relative_to(CSRC)
    return BUILD / (str(rel).replace("/", "__") + ".o")


def _cmd(src: Path) -> list[str]:
    out = str(_obj(src))
    if src.suffix == ".cu":
        return [NVCC, "-std=c++20", "-O3", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC",
                "--expt-relaxed-constexpr", *_DEFS, *INCLUDES, "-c", str(src), "-o", out]
    return ["g++", "-std=c++20", "-O3", "-fPIC", "-Wall", "-Wextra", "-Wno-unused-parameter",
            *INCLUDES, "-c", str(src), "-o", out]


def build(verbose: bool = False, jobs: int | None = None) -> Path:
    BUILD.mkdir(exist_ok=True)
    LIBDIR.mkdir(exist_ok=True)
    cu, cpp = _sources()
    newest_header = max((h.stat().st_mtime for h in _headers()), default=0.0)
    todo = []
    for s in cu + cpp:
        o = _obj(s)
        if not o.exists() or o.stat().st_mtime < max(s.stat().st_mtime, newest_header):
            todo.append(s)

    def run(src):
        cmd = _cmd(src)
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {src}\n{r.stdout}\n{r.stderr}")
        return src

    with cf.ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        list(ex.map(run, todo))
    objs = [str(_obj(s)) for s in cu + cpp]
    if todo or not LIB.exists():
        cmd = [NVCC, "-shared", *ARCH, "-o", str(LIB), *objs, "-lcuda"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed\n{r.stdout}\n{r.stderr}")
    return LIB


def build_sanitized(out: Path, verbose: bool = False) -> Path:
    """The same library with AddressSanitizer + UBSan on every host code path
    (the .cpp files and the host side of the .cu files), for the CPU-side
    checks of tools/asan_check.sh (compute-sanitizer is closed on this GPU
    pool).  Objects and the .so go to `out`, never next to the product."""
    out = Path(out)
    out.mkdir(parents=True, exist_ok=True)
    san = ["-fsanitize=address", "-fsanitize=undefined", "-fno-omit-frame-pointer", "-g"]  # nvcc splits on ","
    cu, cpp = _sources()

    def run(src):
        o = out / (str(src.relative_to(CSRC)).replace("/", "__") + ".o")
        if src.suffix == ".cu":
            cmd = [NVCC, "-std=c++20", "-O1", *ARCH, "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", *INCLUDES,
                   *[x for f in san for x in ("-Xcompiler", f)], "-c", str(src), "-o", str(o)]
        else:
            cmd = ["g++", "-std=c++20", "-O1", "-fPIC", *san, *INCLUDES, "-c", str(src), "-o", str(o)]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {src}\n{r.stdout}\n{r.stderr}")
        return str(o)

    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(run, cu + cpp))
    lib = out / "libcssc_he.so"
    r = subprocess.run([NVCC, "-shared", *ARCH, "-o", str(lib), *objs, "-Xcompiler",
                        "-fsanitize=address", "-Xcompiler", "-fsanitize=undefined"], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed\n{r.stdout}\n{r.stderr}")
    return lib


def build_oracle(verbose: bool = False) -> None:
    """Test-side checkers (oracle/build, oracle/_ref); not part of the product."""
    r = subprocess.run(["make", "-C", str(ROOT / "oracle"), "all"], capture_output=True, text=True)
    if verbose:
        print(r.stdout, r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed\n{r.stdout}\n{r.stderr}")


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
    if "--oracle" in sys.argv:
        build_oracle(verbose=True)
