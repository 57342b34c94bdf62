"""The C ABI library (libfastvol_b200.so) loads without a GPU and exports
every entry point include/fastvol_b200.h declares; without a device the
Python API fails loudly (there is no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "fastvol_b200.h")


def declared():
    src = open(HEADER).read()
    return re.findall(r"FV_API\s+[\w\s\*]+?\b(fv_\w+)\s*\(", src)


@pytest.fixture(scope="module")
def lib():
    from paper_2604_27210_b200 import _build, _native
    _build.build()
    return _native.load()


def test_header_declares_the_batch_entry_points():
    names = declared()
    for n in ("fv_batch_price", "fv_batch_iv", "fv_batch_greeks", "fv_price_greeks", "fv_price_iv"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared():
        assert hasattr(lib, name), name


def test_version_and_device_count(lib):
    assert b"sm_100a" in lib.fv_version()
    n = lib.fv_device_count()
    assert n >= 0


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2604_27210_b200 import _native
    import paper_2604_27210_b200 as fv
    with pytest.raises(_native.NativeUnavailable):
        fv.batch_iv("black", "lbr", ["c"], [100.0], [100.0], [1.0], [0.0], price=[8.0])


def test_sm100a_cubin_in_library():
    import subprocess
    so = os.path.join(REPO, "paper_2604_27210_b200", "libfastvol_b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
