"""Build libfastvol_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2604_27210_b200._build [--force]

Flags that matter for parity: -fmad=false (CPython never fuses a*b+c; the
only fused ops are the explicit __fma_rn calls that mirror glibc's FMA
builds), IEEE fp64 div/sqrt (the CUDA default; no --use_fast_math).
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libfastvol_b200.so")
SOURCES = [os.path.join(CSRC, "fv_kernels.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("fv_quote.h", "fv_libm.h", "fv_tables.h", "fv_fast.h", "fv_consts.h")] + [
    os.path.join(os.path.dirname(HERE), "include", "fastvol_b200.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false",
              "-std=c++17", "-Xptxas", "-v", "-shared", "-Xcompiler", "-fPIC,-fvisibility=hidden",
              "-lcudart"]


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, out=None, defines=()):
    out = out or OUT
    if not force and not _stale(out, DEPS):
        return out
    tmp = out + ".tmp%d" % os.getpid()
    cmd = [NVCC] + NVCC_FLAGS + ["-D" + d for d in defines] + ["-o", tmp] + SOURCES
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    log = os.path.join(os.path.dirname(out), "_build_ptxas.log" if out == OUT else os.path.basename(out) + ".ptxas.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if verbose:
        sys.stdout.write(res.stderr)
    os.replace(tmp, out)
    return out


HOST_SRC = os.path.join(CSRC, "fv_host.cpp")


def host_ext_path():
    import sysconfig
    return os.path.join(HERE, "_fvhost" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_host(force=False):
    """The CPython extension with the batch front end's host loops
    (csrc/fv_host.cpp: flag parsing, status object columns)."""
    import sysconfig
    import numpy
    out = host_ext_path()
    if not force and not _stale(out, [HOST_SRC]):
        return out
    tmp = out + ".tmp%d" % os.getpid()
    cmd = ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread", "-fvisibility=hidden",
           "-I" + sysconfig.get_paths()["include"], "-I" + numpy.get_include(), "-o", tmp, HOST_SRC]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("g++ failed:\n" + res.stdout + res.stderr)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
    print(build_host(force="--force" in sys.argv))
