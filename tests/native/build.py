"""Build the CPU-side test harnesses (host builds of the device headers).
Test infrastructure only."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_build")
FLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC"]
DEPS = [os.path.join(HERE, "..", "..", "paper_2604_27210_b200", "csrc", f)
        for f in ("fv_libm.h", "fv_quote.h", "fv_tables.h", "fv_consts.h", "fv_fast.h")]


def build(name):
    src = os.path.join(HERE, name + ".cpp")
    lib = os.path.join(OUT, "lib" + name + ".so")
    os.makedirs(OUT, exist_ok=True)
    newest = max(os.path.getmtime(p) for p in [src] + DEPS)
    if not os.path.exists(lib) or os.path.getmtime(lib) < newest:
        tmp = lib + ".tmp%d" % os.getpid()
        subprocess.run(["g++"] + FLAGS + ["-o", tmp, src, "-lm"], check=True)
        os.replace(tmp, lib)
    return lib
