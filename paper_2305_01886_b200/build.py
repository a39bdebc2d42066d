"""Build libgk.so (sm_100a only) in-tree with nvcc.

    python -m paper_2305_01886_b200.build [--force]

Flags: -gencode arch=compute_100a,code=sm_100a, -lineinfo for ncu source
pages, and -fmad=false so no multiply-add is contracted into an FMA (every
fp64 expression must round exactly like the reference's CPython floats;
SURVEY §7.3.1).  The glibc-exact exp port uses explicit __fma_rn where the
reference's libm fuses.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libgk.so"
PTX_LIB = PKG / "libgkhost.so"   # host-only native code (g++, no CUDA): PTX front-end, ensemble I/O
PTX_SOURCES = ["gk_ptx.cpp", "gk_ensio.cpp", "gk_featio.cpp"]
PTX_HEADERS = ["gk_ptx.h", "gk_ensio.h", "gk_featio.h"]
CXXFLAGS = ["-O2", "-std=c++17", "-fPIC", "-shared", "-pthread", "-Wall", "-Wextra"]
SOURCES = ["gk_api.cu", "gk_sched.cu", "gk_rf.cu", "gk_rftrain.cu", "gk_corr.cu"]
HEADERS = ["gk_internal.cuh", "gk_exp.h", "gk_exp_table.h", "gk_walk.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
           "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [PKG.parent / "include" / "gk.h"]
    return any(d.stat().st_mtime > t for d in deps)


def build_ptx(force: bool = False) -> Path:
    """libgkhost.so: the native PTX front-end (include/gk_ptx.h) and ensemble
    JSON I/O (include/gk_ensio.h) -- host code, no CUDA."""
    inc = PKG.parent / "include"
    hdrs = [inc / h for h in PTX_HEADERS]
    srcs = [CSRC / s for s in PTX_SOURCES]
    if not force and PTX_LIB.exists() and all(
            d.stat().st_mtime <= PTX_LIB.stat().st_mtime for d in srcs + hdrs):
        return PTX_LIB
    cxx = os.environ.get("CXX") or shutil.which("g++") or "g++"
    tmp = PTX_LIB.with_suffix(".so.tmp")
    cmd = [cxx, *CXXFLAGS, f"-I{inc}", *map(str, srcs), "-o", str(tmp)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(f"g++ failed on {PTX_SOURCES}:\n{r.stdout}{r.stderr}")
    tmp.replace(PTX_LIB)
    return PTX_LIB


def build(force: bool = False, verbose: bool = False) -> Path:
    build_ptx(force)
    if not force and not _stale():
        return LIB
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    objs, procs = [], []
    for src in SOURCES:
        obj = objdir / (Path(src).stem + ".o")
        extra = os.environ.get("GK_NVCC_EXTRA", "").split()
        cmd = [nvcc(), *ARCH, *NVFLAGS, *extra, "-c", str(CSRC / src), "-o", str(obj)]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                            text=True)))
        objs.append(str(obj))
    log = []
    for src, p in procs:
        out, _ = p.communicate()
        log.append(f"== {src}\n{out}")
        if p.returncode:
            raise RuntimeError(f"nvcc failed on {src}:\n{out}")
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(f"link failed:\n{r.stdout}{r.stderr}")
    tmp.replace(LIB)
    (objdir / "ptxas.log").write_text("\n".join(log))
    if verbose:
        print("\n".join(log))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
