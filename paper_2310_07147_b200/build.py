"""Build the sm_100a CUDA library (``_lib/libqft_b200.so``) and the pybind drop-in
module (``qft_engine``) in-tree with explicit nvcc / g++ command lines.

The arithmetic contract matters for parity: ``-fmad=false`` (no FMA contraction,
the reference is built with ``-ffp-contract=off``, CMakeLists.txt:12-14) and no
fast-math.  ``python -m paper_2310_07147_b200.build`` rebuilds when a source is
newer than its output.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(LIBDIR, "libqft_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xptxas", "-O3",
                     "-Xcompiler", "-fPIC,-ffp-contract=off,-O3", "-I" + INCLUDE,
                     "--expt-relaxed-constexpr"]


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build_lib(verbose=False, force=False, extra_flags=(), libdir=LIBDIR):
    """Compile every csrc/*.cu for sm_100a and link libqft_b200.so into `libdir`
    (`extra_flags`/`libdir` build tuning variants, e.g. -DQFT_MIN_CTAS=4)."""
    os.makedirs(libdir, exist_ok=True)
    lib = os.path.join(libdir, "libqft_b200.so")
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(INCLUDE, "*.h"))
    objs = []
    for s in srcs:
        o = os.path.join(libdir, os.path.basename(s)[:-3] + ".o")
        if force or _stale(o, [s] + hdrs):
            _run([NVCC] + NVCC_FLAGS + list(extra_flags) + ["-c", s, "-o", o], verbose)
        objs.append(o)
    if force or _stale(lib, objs):
        _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", lib] + objs, verbose)
    return lib


def build_pyext(verbose=False, force=False):
    """pybind11 module mirroring the reference's ``qft_engine`` quantizer surface."""
    import pybind11

    src = os.path.join(CSRC, "qft_engine_py.cpp")
    if not os.path.exists(src):
        return None
    suffix = sysconfig.get_config_var("EXT_SUFFIX")
    out = os.path.join(PKG, "qft_engine" + suffix)
    deps = [src, LIB, os.path.join(INCLUDE, "qft_b200.h")] + \
        glob.glob(os.path.join(INCLUDE, "qft_b200", "*.hpp"))
    if force or _stale(out, deps):
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off",
               "-I" + INCLUDE, "-I" + pybind11.get_include(),
               "-I" + sysconfig.get_paths()["include"], "-I/usr/local/cuda/include",
               src, "-o", out, "-L" + LIBDIR, "-lqft_b200", "-Wl,-rpath,$ORIGIN/_lib"]
        _run(cmd, verbose)
    return out


def build(verbose=False, force=False):
    build_lib(verbose, force)
    build_pyext(verbose, force)


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
