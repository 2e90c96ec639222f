"""Build libgsv_b200.so (the C-ABI extension) in-tree with nvcc for sm_100a.

No torch extension machinery: the library is plain `extern "C"` over raw
device pointers (include/gsv.h), so it is linked with nvcc directly and
loaded with ctypes.  Incremental: a source is recompiled only when it or a
header is newer than its object.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(CSRC, "build")
LIB = os.path.join(HERE, "libgsv_b200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
          f"-I{INCLUDE}", "--expt-relaxed-constexpr"]
# measurement builds only: extra nvcc flags, e.g. GSV_NVCC_EXTRA="-DGSV_FWD_PREFETCH=1"
COMMON += os.environ.get("GSV_NVCC_EXTRA", "").split()
# Per-file extra flags.  The binning TU must never contract f64 mul+add into
# FMA (bit-exact bounds vs numpy, SURVEY.md §0 finding 1).
EXTRA = {"gsv_bin.cu": ["-fmad=false"]}
SOURCES = ["gsv_capi.cu", "gsv_bin.cu", "gsv_render.cu", "gsv_train.cu", "gsv_metrics.cu",
           "gsv_util.cu", "gsv_diag.cu", "gsv_setup.cu"]


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs += [os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE) if f.endswith(".h")]
    return hs


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, variant: str | None = None,
          defines=()) -> str:
    """Compile and link.  ``variant`` + ``defines`` (measurement builds): the
    objects go to csrc/build_<variant>/ and the library to
    libgsv_b200_<variant>.so, loaded with GSV_LIB=<that path>."""
    global BUILD, LIB, COMMON
    if variant:
        BUILD = os.path.join(CSRC, f"build_{variant}")
        LIB = os.path.join(HERE, f"libgsv_b200_{variant}.so")
        COMMON = COMMON + [f"-D{d}" for d in defines]
    os.makedirs(BUILD, exist_ok=True)
    headers = _headers()
    objs = []
    logs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, [path] + headers):
            cmd = [NVCC, *ARCH, *COMMON, *EXTRA.get(src, []), "-c", path, "-o", obj]
            res = subprocess.run(cmd, capture_output=True, text=True)
            logs.append(res.stdout + res.stderr)
            if res.returncode != 0:
                sys.stderr.write(res.stdout + res.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        logs.append(res.stdout + res.stderr)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc link failed")
    if verbose:
        sys.stdout.write("".join(logs))
    with open(os.path.join(BUILD, "ptxas.log"), "a") as fh:
        fh.write("".join(logs))
    return LIB


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("-v", action="store_true")
    ap.add_argument("-f", action="store_true")
    ap.add_argument("--variant", default=None)
    ap.add_argument("-D", action="append", default=[], help="extra -D (variant builds)")
    a = ap.parse_args()
    print(build(verbose=a.v, force=a.f, variant=a.variant, defines=a.D))
