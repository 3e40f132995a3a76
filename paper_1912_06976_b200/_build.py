"""Build the sm_100a C-ABI library in-tree: paper_1912_06976_b200/libbttb_sm100.so.

Plain nvcc, one object per translation unit, linked as a shared library with
the static CUDA runtime.  ``entries.cu`` is compiled with ``-fmad=false`` (the
entry generators reproduce the reference's rounding; see the file header).
"""
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libbttb_sm100.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", CSRC, "-I", INC,
          "--expt-relaxed-constexpr"]
UNITS = {
    "entries.cu": ["-fmad=false", "-prec-div=true", "-prec-sqrt=true", "-ftz=false"],
    "spectral.cu": ["-Xptxas", "-v"] if os.environ.get("BTTB_PTXAS_VERBOSE") else [],
    "cgls.cu": [],
    "generic.cu": [],
    "hoststage.cu": [],
    "capi.cu": [],
}


def nvcc():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _includes(path, seen=None):
    """Local headers a source includes, transitively (its rebuild dependencies)."""
    import re

    seen = set() if seen is None else seen
    for name in re.findall(r'^#include "([^"]+)"', open(path).read(), re.M):
        for d in (CSRC, INC):
            f = os.path.join(d, name)
            if os.path.exists(f) and f not in seen:
                seen.add(f)
                _includes(f, seen)
    return seen


def build(force=False, verbose=False, variant=None, defines=()):
    """Build the library; ``variant``/``defines`` (development experiments)
    build into build/<variant>/ with extra -D flags instead of in-tree; load
    such a build with BTTB_LIB_PATH=build/<variant>/libbttb_sm100.so."""
    global BUILD, LIB
    if variant:
        BUILD = os.path.join(ROOT, "build", variant)
        LIB = os.path.join(BUILD, "libbttb_sm100.so")
        force = True
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    for unit, flags in UNITS.items():
        src = os.path.join(CSRC, unit)
        obj = os.path.join(BUILD, unit.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, [src] + sorted(_includes(src)) + [__file__]):
            cmd = [nvcc()] + ARCH + COMMON + list(defines) + flags + ["-c", src, "-o", obj]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
    if force or _stale(LIB, objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", LIB] + objs + ["-cudart", "static"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    args = sys.argv[1:]
    var = args[args.index("--variant") + 1] if "--variant" in args else None
    print(build(force="--force" in args, verbose=True, variant=var,
                defines=[a for a in args if a.startswith("-D")]))
